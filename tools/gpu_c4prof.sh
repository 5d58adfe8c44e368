# usage: bash tools/gpu_c4prof.sh TAG -- c4 bench line, ncu launch list of its DCDS call, one
# ncu --set full capture of the main DCDS kernel (each after the command exited 0 without ncu)
TAG=$1; mkdir -p gpurun_out/$TAG
timeout 900 python bench.py --config c4 --steps 20 > gpurun_out/$TAG/bench_c4.json 2> gpurun_out/$TAG/bench_c4.err; echo "bench c4 rc=$?"
CMD="python bench.py --config c4 --steps 2 --warmup 1 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse"
$CMD > gpurun_out/$TAG/plain_c4.json 2> gpurun_out/$TAG/plain_c4.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dcds" --csv \
   --log-file gpurun_out/$TAG/launches_c4.csv $CMD > gpurun_out/$TAG/ncu_launch.log 2>&1; echo "launch rc=$?"
$CMD > gpurun_out/$TAG/plain_c4.json 2> gpurun_out/$TAG/plain_c4.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dcds_kernel -s 1 -c 1 \
   -o gpurun_out/$TAG/prof_c4 $CMD > gpurun_out/$TAG/ncu_c4.log 2>&1; echo "full c4 rc=$?"
