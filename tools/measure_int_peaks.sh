# usage: bash tools/measure_int_peaks.sh  -- VABSDIFF4 / IDP.4A / SHF issue rates on the GPU
# (8 independent chains per thread, full occupancy) -> gpurun_out/int_peaks.json; the bench
# roofline reads the committed copy profiles/int_peaks.json
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_peaks tools/int_peaks.cu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 ./tools/int_peaks > gpurun_out/int_peaks.json; echo "int_peaks rc=$?"
cat gpurun_out/int_peaks.json
