O=gpurun_out/s2z6; mkdir -p $O
timeout 900 python -m pytest -q -x -m gpu tests/test_compat_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 900 python bench.py --no-cpu --no-north-star > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.loads([l for l in open('$O/bench.json') if l.startswith('{')][-1]); print(d['e2e']['value'], d['e2e_numpy_dropin'])" > $O/summary.txt
