# usage: bash tools/ncu_one.sh <tag> <config> [env assignments...]  -- one ncu --set full capture of the search kernel
TAG=$1; CFG=$2; shift 2
env "$@" timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dcds -s 1 -c 1 \
   -o gpurun_out/prof_$TAG python bench.py --config $CFG --steps 2 --warmup 1 --no-fs --no-e2e --no-cpu > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
