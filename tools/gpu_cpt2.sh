TAG=$1
mkdir -p gpurun_out/$TAG
timeout 900 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__registers_per_thread,sm__maximum_warps_per_active_cycle_pct --clock-control none -k regex:dcds --csv --log-file gpurun_out/$TAG/ncu_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-fs --no-e2e --no-cpu --no-cmp --no-mcsse > gpurun_out/$TAG/ncu.log 2>&1
echo rc=$?
python - <<'PY'
import csv,sys
rows=list(csv.reader(open('gpurun_out/'+sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/cpt2/ncu_c4.csv')))
PY
grep -E "dcds" gpurun_out/$TAG/ncu_c4.csv | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}' | cut -c1-200 | head -40
