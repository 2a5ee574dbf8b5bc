# new GPU tests + per-shard-size DRAM traffic (ncu) of the persistent launch
mkdir -p gpurun_out/traffic
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_compat_gpu.py tests/test_chain_gpu.py tests/test_dynamics_gpu.py tests/test_controllers_gpu.py > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
run() {  # config n
  timeout 600 ncu --metrics $M --clock-control none -k regex:stream_kernel --launch-skip 3 --launch-count 1 --csv \
    python bench.py --config $1 --n $2 --steps 20 --warmup 3 --no-cpu --no-fused --no-e2e --no-north-star \
    > gpurun_out/traffic/$1@$2.csv 2> gpurun_out/traffic/$1@$2.err
}
for n in 4194304 2097152 1048576 524288; do run cfg2 $n; done
for n in 16777216 8388608 4194304 2097152; do run cfg3 $n; done
for n in 1048576 524288 262144 131072; do run cfg1 $n; done
for n in 8388608 4194304 2097152 1048576; do run cfg4 $n; done
