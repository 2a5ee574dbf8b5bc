mkdir -p gpurun_out; rm -f gpurun_out/m_forest.txt
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py > gpurun_out/pytest_m.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_m.log
for cw in 30 60 100 200 400; do
  timeout 600 python bench.py --config forest --steps 100 --no-cpu --no-e2e --clear-walk-cm $cw 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('walk', $cw, round(d['ms_per_step']*1e3,1), d['collision_tests']['fraction'])" >> gpurun_out/m_forest.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"world_|scene_fix" --launch-skip 12 --launch-count 12 --csv python bench.py --config forest --steps 5 --warmup 3 --no-cpu --no-e2e --no-fused > gpurun_out/m_forest_ncu.csv 2>/dev/null
