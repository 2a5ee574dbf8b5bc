# Scene / camera round: GPU tests of the new path, world regression, render probe.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_scene_gpu.py -q -x > gpurun_out/scene_tests.log 2>&1; echo "scene rc=$?" >> gpurun_out/scene_tests.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python tools/gpu_render.py > gpurun_out/render.json 2> gpurun_out/render.err; echo "render rc=$?"
timeout 300 python tools/gpu_render.py --envs 256 --width 64 --height 48 > gpurun_out/render_small.json 2>> gpurun_out/render.err; echo "render small rc=$?"
