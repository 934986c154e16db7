mkdir -p gpurun_out; : > gpurun_out/exp_l2.log
for h in 0 1 0 1; do FORGE_SCAN_L2HINT=$h timeout 300 python tools/probe.py scan | sed "s/^/hint=$h /" >> gpurun_out/exp_l2.log 2>&1; done
FORGE_SCAN_L2HINT=1 timeout 300 python tools/probe.py scan --check | sed "s/^/hint=1 check /" >> gpurun_out/exp_l2.log 2>&1
