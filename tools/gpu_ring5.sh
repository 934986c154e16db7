mkdir -p gpurun_out
for i in 1 2 3 4; do for R in 28 12 13 29; do
  FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 45 python tools/probe.py scan > /tmp/o.log 2>&1
  echo "ring=$R rc=$? $(tail -c 200 /tmp/o.log)" >> gpurun_out/ring5.log
done; done
exit 0
