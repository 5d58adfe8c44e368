set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "not c4" 2>&1 | tail -5
for G in 4 8; do for T in 16,8 32,8 16,4; do
  ME_G=$G ME_TILE=$T timeout 300 python bench.py --steps 10 --warmup 3 --no-fs --no-e2e --no-cpu > gpurun_out/tune_c3_${G}_${T}.json 2>&1
  echo "G=$G T=$T $(python -c "import json;d=json.load(open('gpurun_out/tune_c3_${G}_${T}.json'));print(d['ms_per_step'], d['value'], d['roofline']['frac'])")"
done; done
bash tools/gpu_prof.sh ${1:-r1c} c3
