mkdir -p gpurun_out
for op in 0 11; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_lag -s 2 -c 1 -o /tmp/lag_$op python tools/one_kernel.py scan $op > gpurun_out/ncu_lag_$op.log 2>&1
ncu -i /tmp/lag_$op.ncu-rep --page raw --csv > gpurun_out/lag_${op}_raw.csv 2>/dev/null
ncu -i /tmp/lag_$op.ncu-rep --page details --csv > gpurun_out/lag_${op}_details.csv 2>/dev/null
ncu -i /tmp/lag_$op.ncu-rep --page source --csv > gpurun_out/lag_${op}_source.csv 2>/dev/null
done
