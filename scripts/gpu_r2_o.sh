mkdir -p gpurun_out; rm -f gpurun_out/o_forest.txt
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py -k "clearance or forest" > gpurun_out/pytest_o.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_o.log
for ex in 0 1; do for cw in 30 100 200; do
  timeout 600 python bench.py --config forest --steps 100 --no-cpu --no-e2e --clear-walk-cm $cw --clear-exact $ex 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exact', $ex, 'walk', $cw, round(d['ms_per_step']*1e3,1), round(d['collision_tests']['fraction'],4), round(d['roofline']['frac'],3))" >> gpurun_out/o_forest.txt
done; done
