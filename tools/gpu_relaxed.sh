mkdir -p gpurun_out
timeout 300 python tools/probe.py scan --check > gpurun_out/relaxed.log 2>&1
for L in libforge_old.so libforge.so; do FORGE_LIB=$L timeout 300 python tools/probe_small.py >> gpurun_out/relaxed.log 2>&1; done
for op in 12 10 11 0; do timeout 60 python tools/hang_probe.py $op 400 27 >> gpurun_out/relaxed.log 2>&1; done
timeout 120 python tools/hang_probe2.py 40 28 >> gpurun_out/relaxed.log 2>&1
for op in 0 11; do timeout 120 python tools/trace_lag.py $op 28 >> gpurun_out/relaxed.log 2>&1; done
timeout 3000 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/pytest_relaxed.log 2>&1; echo rc=$? >> gpurun_out/pytest_relaxed.log
exit 0
