# Scratch GPU experiment (development; overwritten per experiment)
mkdir -p gpurun_out; : > gpurun_out/exp.log
for b in 2 3 4 5 3 4; do FORGE_GEMV_BLOCKS_PER_SM=$b timeout 120 python tools/probe.py matrix | tail -1 | sed "s/^/bps=$b /" >> gpurun_out/exp.log 2>&1; done
