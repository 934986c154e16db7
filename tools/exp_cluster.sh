mkdir -p gpurun_out; : > gpurun_out/exp_ord.log
timeout 300 python tools/probe.py ordered >> gpurun_out/exp_ord.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ordered or sharded or c5 or mapreduce or noncommut" --timeout 600 -p no:randomly > gpurun_out/pytest_ord.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_ord.log
