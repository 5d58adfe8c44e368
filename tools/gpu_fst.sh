# usage: bash tools/gpu_fst.sh TAG "threads..." -- c3 FS throughput (64 pairs) per ME_FS_THREADS
TAG=$1
mkdir -p gpurun_out/$TAG
for t in $2; do
  ME_FS_THREADS=$t timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse --fs-pairs 64 > gpurun_out/$TAG/b_$t.json 2>gpurun_out/$TAG/b_$t.err
  python -c "import json;d=json.load(open('gpurun_out/$TAG/b_$t.json'))['fullsearch'];print('$t', round(d['ms'],3), round(d['alu_frac'],3))"
done
