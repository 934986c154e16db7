mkdir -p gpurun_out
for R in 28 12 24 8 28; do
  echo "ring=$R" >> gpurun_out/ring4.log
  FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 60 python tools/probe.py scan >> gpurun_out/ring4.log 2>&1
  echo "rc=$?" >> gpurun_out/ring4.log
done
exit 0
