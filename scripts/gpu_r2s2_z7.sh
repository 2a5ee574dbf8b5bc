# the driver's own invocations (round-1 BENCH command line), ours and the reference arm
O=gpurun_out/s2z7; mkdir -p $O
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "rc=$?" >> $O/rc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_trun.json 2> $O/bench_trun.err; echo "rc=$?" >> $O/rc.txt
