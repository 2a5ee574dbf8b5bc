# run-to-run spread on one box: 5 x default bench (cfg2 + north star), 5 x cfg3 at 2^21 (the
# north star's per-GPU shard), 5 x forest
O=gpurun_out/s2v; mkdir -p $O
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-cpu --no-e2e > $O/default_$i.json 2>/dev/null
  timeout 600 python bench.py --config cfg3 --n 2097152 --no-cpu > $O/cfg3_2m_$i.json 2>/dev/null
  timeout 600 python bench.py --config forest --no-cpu > $O/forest_$i.json 2>/dev/null
done
