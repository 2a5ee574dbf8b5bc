O=gpurun_out/s2zj; mkdir -p $O
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -p no:randomly > $O/pytest_$i.txt 2>&1; echo "rc=$?" >> $O/pytest_$i.txt
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
