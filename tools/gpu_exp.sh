mkdir -p gpurun_out
timeout 300 python tools/debug_mutant.py > gpurun_out/mutant.log 2>&1
timeout 300 python tools/probe.py scan > gpurun_out/probe.log 2>&1
timeout 300 python tools/probe.py matrix >> gpurun_out/probe.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_semantics.py -q --timeout 600 -p no:randomly > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
