mkdir -p gpurun_out; : > gpurun_out/exp_e.log
timeout 300 python tools/probe.py scan --check >> gpurun_out/exp_e.log 2>&1
FORGE_SCAN_EARLY=0 timeout 300 python tools/probe.py scan >> gpurun_out/exp_e.log 2>&1
FORGE_SCAN_LOOKBACK=99 timeout 300 python tools/probe.py scan >> gpurun_out/exp_e.log 2>&1
timeout 300 python tools/trace_scan.py 0 28 2>&1 | grep -v "^  \|^ }" >> gpurun_out/exp_e.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "scan" --timeout 300 -p no:randomly > gpurun_out/pytest_scan.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_scan.log
