for t in 64 128 256; do
for c in c3 c4; do
ME_MC_THREADS=$t timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp > gpurun_out/mc_$c.json 2>/dev/null
echo "$t $c $(python -c "import json;d=json.load(open('gpurun_out/mc_$c.json'))['mc_sse_standalone'];print(round(d['ms'],4), round(d['frac_hbm'],3))")"
done; done
