# Scratch GPU experiment (development; overwritten per experiment)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench_final.log
