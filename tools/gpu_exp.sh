# Scratch GPU experiment (development; overwritten per experiment)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown --no-sharded-scan > gpurun_out/bench_ncu.log 2>&1
