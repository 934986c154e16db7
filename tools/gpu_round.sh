# Full measurement pass on one B200: GPU tests, bench, ncu launch list, ncu full captures (exported to CSV).
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:randomly > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
fi
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref_rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown --no-sharded-scan > gpurun_out/bench_ncu.log 2>&1
for k in "mapreduce:1:mapreduce_kernel" "scan:0:scan_smem_kernel" "gevm:32:gevm_cols_kernel" "gemv:32:gemv_kernel" "copy:0:vcopy_kernel"; do
  args=$(echo $k | cut -d: -f1); op=$(echo $k | cut -d: -f2); pat=$(echo $k | cut -d: -f3)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 1 -c 1 -o /tmp/full_$args python tools/one_kernel.py $args $op > gpurun_out/ncu_$args.log 2>&1
  ncu -i /tmp/full_$args.ncu-rep --page raw --csv > gpurun_out/full_${args}_raw.csv 2>/dev/null
  ncu -i /tmp/full_$args.ncu-rep --page details --csv > gpurun_out/full_${args}_details.csv 2>/dev/null
  ncu -i /tmp/full_$args.ncu-rep --page source --csv > gpurun_out/full_${args}_source.csv 2>/dev/null
done
cp /tmp/full_mapreduce.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out; ls -la gpurun_out
