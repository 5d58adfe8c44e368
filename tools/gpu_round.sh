# usage: bash tools/gpu_round.sh <tag>  -- the round's evidence: default bench lines (c3, c4),
# the ncu launch list of the default command, one ncu --set full capture of the DCDS kernel per
# config (each ncu run only after the same command exited 0 without ncu)
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
timeout 900 python bench.py > gpurun_out/$TAG/bench_c3.json 2> gpurun_out/$TAG/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c4 --steps 20 > gpurun_out/$TAG/bench_c4.json 2> gpurun_out/$TAG/bench_c4.err; echo "bench c4 rc=$?"
CMD="python bench.py --steps 2 --warmup 1"
$CMD > gpurun_out/$TAG/plain_launch.json 2> gpurun_out/$TAG/plain_launch.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dcds_kernel|fs_kernel|mc_sse|quality|bma" -c 400 --csv \
   --log-file gpurun_out/$TAG/launches_c3.csv $CMD > gpurun_out/$TAG/ncu_launch.log 2>&1; echo "launch rc=$?"
for c in c3 c4; do
  CMD="python bench.py --config $c --steps 2 --warmup 1 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse"
  $CMD > gpurun_out/$TAG/plain_$c.json 2> gpurun_out/$TAG/plain_$c.err && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dcds_kernel -s 1 -c 1 \
     -o gpurun_out/$TAG/prof_$c $CMD > gpurun_out/$TAG/ncu_$c.log 2>&1
  echo "full $c rc=$?"
done
