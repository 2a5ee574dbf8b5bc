# ncu evidence for the obstacle World.step and the depth camera (exported on the box)
mkdir -p gpurun_out
B="python bench.py --config forest --steps 10 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step_kernel -s 5 -c 1 -o gpurun_out/forest_p $B > gpurun_out/ncu_forest.log 2>&1; echo "forest rc=$?"
B="python bench.py --config render --steps 3 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/render_p $B > gpurun_out/ncu_render.log 2>&1; echo "render rc=$?"
for c in forest render; do
  ncu -i gpurun_out/${c}_p.ncu-rep --page details > gpurun_out/${c}_details.txt 2>&1
  ncu -i gpurun_out/${c}_p.ncu-rep --page raw --csv > gpurun_out/${c}_raw.csv 2>&1
  rm -f gpurun_out/${c}_p.ncu-rep
done
