# usage: bash tools/gpu_fssw.sh TAG -- FS parity tests; c3 FS (32 pairs) with the column sweep
# (default) / the chunked kernel (ME_FS_SWEEP=0), thread counts
TAG=$1; mkdir -p gpurun_out/$TAG
[ -n "$3" ] && timeout 600 python -m pytest tests -m gpu -x -q -k "fs or full or fuzz" > gpurun_out/$TAG/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/$TAG/tests.log
for e in $2; do
  n=$(echo "$e" | tr ' =,/' '____')
  env $e timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/fs_$n.json 2>/dev/null
  echo "[$e] $(python -c "import json;d=json.load(open('gpurun_out/$TAG/fs_$n.json'))['fullsearch'];print(round(d['ms'],4), round(d['alu_frac'],4))" 2>&1 | tail -1)"
done
