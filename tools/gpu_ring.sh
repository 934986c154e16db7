# lagged scan with ring row prefixes: timing + parity (development)
mkdir -p gpurun_out
timeout 300 python tools/probe.py scan --check > gpurun_out/ring_probe.log 2>&1
timeout 300 python tools/probe.py scan >> gpurun_out/ring_probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "lag or stress or scan" -p no:randomly > gpurun_out/pytest_ring.log 2>&1; echo rc=$? >> gpurun_out/pytest_ring.log
