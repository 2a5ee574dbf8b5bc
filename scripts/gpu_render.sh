mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_scene_gpu.py -q -x > gpurun_out/scene_tests.log 2>&1; echo "scene rc=$?" >> gpurun_out/scene_tests.log
for M in 2 1; do
  FS_RENDER_MINB=$M timeout 300 python tools/gpu_render.py > gpurun_out/render_m$M.json 2>> gpurun_out/render.err
  FS_RENDER_MINB=$M timeout 300 python tools/gpu_render.py --depth 5 > gpurun_out/render_d5_m$M.json 2>> gpurun_out/render.err
done
echo done
