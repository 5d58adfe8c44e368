# usage: bash tools/measure_int_peaks.sh  -- VABSDIFF4 / IDP.4A / SHF issue rates (profiles/int_peaks.json)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 ./tools/int_peaks > gpurun_out/int_peaks.json; echo "int_peaks rc=$?"
cat gpurun_out/int_peaks.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c4" 2>&1 | tail -30; echo "pytest rc=$?"
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
