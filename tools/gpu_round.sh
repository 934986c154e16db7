# Full measurement pass on one B200: GPU tests, bench, ncu launch list, ncu full captures.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:randomly > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref_rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
for k in "mapreduce 1:mapreduce_kernel" "scan 0:scan_smem_kernel" "gevm 32:gevm_kernel" "gemv 32:gemv_kernel"; do
  set -- $k; args=${1}; what=${2%%:*}; pat=${2##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 1 -c 1 -o gpurun_out/full_$args python tools/one_kernel.py $args $what > gpurun_out/ncu_$args.log 2>&1
done
ls -la gpurun_out
