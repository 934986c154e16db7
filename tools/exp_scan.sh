mkdir -p gpurun_out; : > gpurun_out/probe.log
for lb in 0 1 2 4; do for sw in 2 32; do
  FORGE_SCAN_LOOKBACK=$lb FORGE_SCAN_STATE_WORDS=$sw python tools/probe.py scan | sed "s/^/lb=$lb sw=$sw /" >> gpurun_out/probe.log 2>&1
done; done
cat gpurun_out/probe.log
