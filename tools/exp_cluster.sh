mkdir -p gpurun_out; : > gpurun_out/exp_c1.log
timeout 300 python tools/probe.py c1g --check >> gpurun_out/exp_c1.log 2>&1
timeout 300 python tools/probe.py c1 >> gpurun_out/exp_c1.log 2>&1
timeout 300 python tools/probe.py scan >> gpurun_out/exp_c1.log 2>&1
