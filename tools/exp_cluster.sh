mkdir -p gpurun_out; : > gpurun_out/exp_g.log
for b in 3 4 6; do FORGE_GEMV_BLOCKS_PER_SM=$b timeout 120 python tools/probe.py matrix | tail -1 | sed "s/^/bps=$b /" >> gpurun_out/exp_g.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -k "matvec or vecmat or gevm or gemv or matrix or mapreduce_2d" --timeout 300 -p no:randomly > gpurun_out/pytest_mat.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_mat.log
