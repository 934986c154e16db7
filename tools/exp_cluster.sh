mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stress.py tests/test_gpu_primitives.py -m gpu -q -x -k "stress or sanitizer or plans" --timeout 900 -p no:randomly --durations=5 > gpurun_out/pytest_stress.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_stress.log
