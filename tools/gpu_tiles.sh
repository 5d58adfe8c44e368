# usage: bash tools/gpu_tiles.sh TAG "NW,TX,TY ..." -- c3 DCDS kernel ms per (ME_NW, ME_TILE)
TAG=$1
mkdir -p gpurun_out/$TAG
for g in $2; do
  nw=${g%%,*}; t=${g#*,}
  ME_NW=$nw ME_TILE=$t timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/b_$nw_$t.json 2>gpurun_out/$TAG/b.err
  python -c "import json;d=json.load(open('gpurun_out/$TAG/b_$nw_$t.json'));print('NW=$nw tile=$t', round(d['kernel_ms_mean'],4))" 2>&1 | tail -1
done
