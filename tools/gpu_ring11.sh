mkdir -p gpurun_out
for L in libforge_old.so libforge.so libforge_old.so libforge.so; do FORGE_LIB=$L timeout 300 python tools/probe.py scan >> gpurun_out/oldnew.log 2>&1; done
for op in 12 10 11; do timeout 60 python tools/hang_probe.py $op 400 27 >> gpurun_out/oldnew.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x -k "lag or stress" -p no:randomly > gpurun_out/pytest_ring11.log 2>&1; echo rc=$? >> gpurun_out/pytest_ring11.log
exit 0
