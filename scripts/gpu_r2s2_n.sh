O=gpurun_out/s2n; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python tools/gpu_cfg3_tune.py > $O/tune.txt 2>&1
timeout 300 python tools/gpu_cfg3_tune.py >> $O/tune.txt 2>&1
FS_BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 100 --warmup 5 --no-cpu --no-e2e \
  > $O/bench_dist1.json 2> $O/bench_dist1.err
