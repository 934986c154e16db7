bash tools/gpu_quick.sh
timeout 300 python tools/debug_mutant.py > gpurun_out/mutant.log 2>&1; echo "mutant_rc=$?" >> gpurun_out/mutant.log
FORGE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench2_rc=$?" >> gpurun_out/bench2.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "benchref_rc=$?" >> gpurun_out/bench_ref.log
