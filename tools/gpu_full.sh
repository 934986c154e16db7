# full check: smoke, probes, hang watchdogs, whole GPU suite, bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/full_smoke.log
timeout 300 python tools/probe_ops.py > gpurun_out/full.log 2>&1
timeout 300 python tools/probe.py scan --check >> gpurun_out/full.log 2>&1
for op in 12 10 11 0; do timeout 60 python tools/hang_probe.py $op 400 27 >> gpurun_out/full.log 2>&1; done
timeout 120 python tools/hang_probe2.py 40 28 >> gpurun_out/full.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/pytest_full.log 2>&1; echo rc=$? >> gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
exit 0
