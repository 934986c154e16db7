mkdir -p gpurun_out
timeout 120 ./tools/probe_lag > gpurun_out/lag.log 2>&1
for i in 11 12 13 14 15; do
timeout 120 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -s 3 -c 1 --csv ./tools/probe_lag $i >> gpurun_out/lag_ncu.csv 2>&1
done
