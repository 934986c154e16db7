# Scratch GPU experiment (development; overwritten per experiment): run with
#   gpurun -- bash tools/gpu_exp.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "scan" --timeout 900 -p no:randomly > gpurun_out/pytest_scan.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_scan.log
timeout 300 python tools/probe.py scan > gpurun_out/exp_wide.log 2>&1
