# usage: bash tools/gpu_fsprof.sh TAG -- one ncu --set full capture of the FS kernel at c3 and c4
# (bench's fullsearch leg, 32 pairs; each after the same command exited 0 without ncu)
TAG=$1; mkdir -p gpurun_out/$TAG
for c in c3 c4; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse --fs-pairs 32"
  $CMD > gpurun_out/$TAG/plain_fs_$c.json 2> /dev/null && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fs_kernel -s 1 -c 1 \
     -o gpurun_out/$TAG/prof_fs_$c $CMD > gpurun_out/$TAG/ncu_fs_$c.log 2>&1
  echo "fs $c rc=$?"
done
