mkdir -p gpurun_out; : > gpurun_out/exp_uf8.log
timeout 300 python tools/probe.py mapreduce --check >> gpurun_out/exp_uf8.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "uf8 or UF8 or mapreduce" --timeout 600 -p no:randomly > gpurun_out/pytest_uf8.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_uf8.log
