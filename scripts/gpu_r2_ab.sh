# forest: clearance-walk radius sweep (FS_TUNE_CLEAR_WALK_CM) on the bench
mkdir -p gpurun_out/r2ab
for cm in 40 70 100 150; do
  timeout 600 python bench.py --config forest --no-cpu --no-e2e --clear-walk-cm $cm > gpurun_out/r2ab/walk_$cm.json 2>/dev/null
done
