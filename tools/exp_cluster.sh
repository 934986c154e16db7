mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gevm_cols_kernel -s 1 -c 1 -o /tmp/full_gevm python tools/one_kernel.py gevm 32 > gpurun_out/ncu_gevm.log 2>&1
ncu -i /tmp/full_gevm.ncu-rep --page raw --csv > gpurun_out/full_gevm_raw.csv 2>/dev/null
ncu -i /tmp/full_gevm.ncu-rep --page details --csv > gpurun_out/full_gevm_details.csv 2>/dev/null
