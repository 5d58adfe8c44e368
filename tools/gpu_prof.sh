# usage: bash tools/gpu_prof.sh <tag> <config>
set -x
TAG=${1:-r1}; CFG=${2:-c3}
CMD="python bench.py --config $CFG --steps 3 --warmup 1 --no-fs --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain_$TAG.json 2> gpurun_out/plain_$TAG.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dcds_kernel|fs_kernel|mc_sse" -c 40 --csv \
   --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dcds -s 1 -c 1 \
   -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
