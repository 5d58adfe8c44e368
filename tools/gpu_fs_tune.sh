# usage: bash tools/gpu_fs_tune.sh "<cfg> <threads> [tile] [split]" ...  -- FS launch sweeps
for spec in "$@"; do
  set -- $spec
  out=gpurun_out/fst_$1_$2_${3:-d}_${4:-d}.json
  env ME_FS_THREADS=$2 ${3:+ME_FS_TILE=$3} ${4:+ME_FS_SPLIT=$4} timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp > $out 2>/dev/null
  echo "$spec $(python -c "import json;d=json.load(open('$out'))['fullsearch'];print(round(d['ms'],4), round(d['alu_frac'],3))" 2>&1 | tail -1)"
done
