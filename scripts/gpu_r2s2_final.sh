# round-2 session-2 final pass (one box): traffic captures first (bench reads
# profiles/traffic.json), then the GPU suite, smoke, every bench line (ours +
# reference), a one-rank NCCL run of the multi-GPU path, launch list, ncu captures
O=gpurun_out/s2z
mkdir -p $O/traffic
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,memory.total --format=csv > $O/gpu.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
# forest: the three kernels of one steady-state step (step 111 of a fresh world)
timeout 600 ncu --metrics $M --clock-control none --profile-from-start off --csv \
  python tools/forest_step_for_ncu.py > $O/traffic/forest@2097152_steps.csv 2> $O/traffic/forest.err
# cfg4: the bench's persistent launch again (round-2 capture read 1.17 x algorithmic)
timeout 600 ncu --metrics $M --clock-control none -k regex:stream_kernel --launch-skip 3 --launch-count 1 --csv \
  python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu --no-fused --no-e2e --no-north-star \
  > $O/traffic/cfg4@8388608.csv 2> $O/traffic/cfg4.err
timeout 600 ncu --metrics $M --clock-control none -k regex:stream_kernel --launch-count 8 --csv \
  python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu --no-fused --no-e2e --no-north-star \
  > $O/traffic/cfg4_first8.csv 2> /dev/null
for f in $O/traffic/forest@2097152_steps.csv $O/traffic/cfg4@8388608.csv; do
  if grep -q dram__bytes_write "$f"; then cp "$f" profiles/raw/r2_traffic/; fi
done
python tools/traffic_table.py profiles/raw/r2_traffic > $O/traffic.json && cp $O/traffic.json profiles/traffic.json
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for c in cfg0 cfg1 cfg3 cfg4 world vecenv forest render; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
for c in forest render cfg3; do
  timeout 600 python bench.py --impl reference --config $c > $O/bench_ref_$c.json 2> $O/bench_ref_$c.err
done
# the multi-GPU code path (NCCL communicator, barriers, max over ranks, the
# statistics all-reduce) as one rank under torchrun
FS_BENCH_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 200 --warmup 5 --no-cpu \
  > $O/bench_dist1.json 2> $O/bench_dist1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-fused --north-star-steps 20 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 3 --launch-count 1 \
  -o $O/cfg2_full python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-fused --no-north-star > $O/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 3 --launch-count 1 \
  -o $O/cfg3_full python bench.py --config cfg3 --n 2097152 --steps 20 --warmup 3 --no-cpu --no-e2e --no-fused > $O/ncu_cfg3.log 2>&1
echo done > $O/DONE
