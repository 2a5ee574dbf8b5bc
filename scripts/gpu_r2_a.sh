# round 2: new parity tests + kernel memory-model changes, then a quick bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
    tests/test_controllers_gpu.py tests/test_dynamics_gpu.py tests/test_chain_gpu.py \
    tests/test_scene_gpu.py::test_autoreset_placement_failure_raises > gpurun_out/pytest_new.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_new.log
for c in cfg2 cfg3; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-fused > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
