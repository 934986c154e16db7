mkdir -p gpurun_out; : > gpurun_out/exp_lb.log
timeout 300 python tools/probe.py scan --check >> gpurun_out/exp_lb.log 2>&1
timeout 300 python tools/trace_scan.py >> gpurun_out/exp_lb.log 2>&1
FORGE_SCAN_LOOKBACK=99 timeout 300 python tools/probe.py scan >> gpurun_out/exp_lb.log 2>&1
