# cfg2 at the per-GPU shard sizes of 1/2/4/8-GPU strong scaling (2^22 total), one GPU each
O=gpurun_out/s2z5; mkdir -p $O
for n in 4194304 2097152 1048576 524288; do
  timeout 600 python bench.py --n $n --no-cpu --no-e2e --no-north-star > $O/cfg2_$n.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('$O/cfg2_$n.json') if l.startswith('{')][-1]); print($n, '%.4g'%d['value'], round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), d['config']['l2'][:60], d['persistent_launch']['ms_per_step']*1e3, d['per_step_launches']['ms_per_step']*1e3)" >> $O/summary.txt
done
