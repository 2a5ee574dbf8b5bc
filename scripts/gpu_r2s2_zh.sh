O=gpurun_out/s2zh; mkdir -p $O
timeout 900 python tools/chain_stress.py 20 > $O/stress_small.txt 2>&1
timeout 900 python tools/chain_stress_big.py 4 > $O/stress_big.txt 2>&1
