O=gpurun_out/s2zi; mkdir -p $O
for nc in 0 16 0 16; do
  timeout 600 python bench.py --config cfg4 --no-cpu --ncw $nc > $O/cfg4_$nc.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('$O/cfg4_$nc.json') if l.startswith('{')][-1]); print('ncw', $nc, round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3), d['persistent_launch']['ms_per_step']*1e3, d['per_step_launches']['ms_per_step']*1e3)" >> $O/summary.txt
done
