O=gpurun_out/s2z3; mkdir -p $O
timeout 180 python -m pytest -q -x -m gpu tests/test_fleet_gpu.py -k control_only -p no:cacheprovider > $O/pytest_ctl.txt 2>&1; echo "rc=$?" >> $O/pytest_ctl.txt
nvidia-smi --query-gpu=name,utilization.gpu --format=csv >> $O/pytest_ctl.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python tools/gpu_cfg3_tune.py > $O/tune.txt 2>&1
