# compat test, launch-shape sweep over shard sizes, per-step traffic, cfg3 full ncu with source
mkdir -p gpurun_out/traffic gpurun_out/sweep
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_compat_gpu.py > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g.log
sw() { timeout 300 python bench.py --config $1 --n $2 --steps 200 --warmup 5 --no-cpu --no-fused --no-e2e --no-north-star > gpurun_out/sweep/$1@$2.json 2>/dev/null; }
for n in 4194304 2097152 1048576 524288; do sw cfg2 $n; done
for n in 16777216 8388608 4194304 2097152; do sw cfg3 $n; done
for n in 1048576 524288 262144 131072; do sw cfg1 $n; done
for n in 8388608 4194304 2097152 1048576; do sw cfg4 $n; done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
st() {
  timeout 600 ncu --metrics $M --clock-control none -k regex:stream_kernel --launch-skip 7 --launch-count 1 --csv \
    python bench.py --config $1 --n $2 --steps 20 --warmup 3 --no-cpu --no-fused --no-e2e --no-north-star \
    > gpurun_out/traffic/$1@$2_steps.csv 2> gpurun_out/traffic/$1@$2_steps.err
}
for n in 2097152 1048576 524288; do st cfg2 $n; done
for n in 4194304 2097152; do st cfg3 $n; done
for n in 524288 262144 131072; do st cfg1 $n; done
for n in 2097152 1048576; do st cfg4 $n; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 3 --launch-count 1 \
   -o gpurun_out/r2_cfg3_full python bench.py --config cfg3 --n 2097152 --steps 20 --warmup 3 --no-cpu --no-fused --no-e2e > gpurun_out/ncu_cfg3.log 2>&1
