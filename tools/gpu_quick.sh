# Quick GPU pass (development): smoke, scan/mapreduce probes, tests, bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/probe.py scan > gpurun_out/probe.log 2>&1
timeout 300 python tools/probe.py matrix >> gpurun_out/probe.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 -p no:randomly ${PYTEST_ARGS:-} > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
if [ "${SKIP_BENCH:-0}" != "1" ]; then
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
fi
