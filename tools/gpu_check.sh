# quick check after a scan change: probe (+oracle check), hang watchdogs, scan/lag/stress tests, bench
mkdir -p gpurun_out
timeout 300 python tools/probe.py scan --check > gpurun_out/check.log 2>&1
for op in 12 10 11 0; do timeout 60 python tools/hang_probe.py $op 400 27 >> gpurun_out/check.log 2>&1; done
timeout 120 python tools/hang_probe2.py 40 28 >> gpurun_out/check.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -k "lag or stress or scan" -p no:randomly > gpurun_out/pytest_check.log 2>&1; echo rc=$? >> gpurun_out/pytest_check.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_check.log 2>&1
timeout 300 python tools/probe_small.py >> gpurun_out/check.log 2>&1
timeout 300 python tools/probe_cyclic.py >> gpurun_out/check.log 2>&1
exit 0
