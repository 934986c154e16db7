mkdir -p gpurun_out
timeout 300 python tools/debug_mutant.py > gpurun_out/mutant.log 2>&1
timeout 900 python bench.py --steps 5 > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
FORGE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --no-breakdown > gpurun_out/bench2.log 2>&1; echo "bench2_rc=$?" >> gpurun_out/bench2.log
