mkdir -p gpurun_out/fsp
for n in 4 16 64 239; do
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse --fs-pairs $n > gpurun_out/fsp/b_$n.json 2>gpurun_out/fsp/b_$n.err
python -c "import json;d=json.load(open('gpurun_out/fsp/b_$n.json'))['fullsearch'];print($n, round(d['ms'],3), round(d['alu_frac'],3))"
done
for n in 2 8; do
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-cmp --no-mcsse --fs-pairs $n > gpurun_out/fsp/c4_$n.json 2>gpurun_out/fsp/c4_$n.err
python -c "import json;d=json.load(open('gpurun_out/fsp/c4_$n.json'))['fullsearch'];print('c4', $n, round(d['ms'],3), round(d['alu_frac'],3))"
done
