mkdir -p gpurun_out
./tools/context_bench > gpurun_out/context.json 2> gpurun_out/context.err
FORGE_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --elems 268435456 > gpurun_out/bench2.log 2>&1; echo "bench2_rc=$?" >> gpurun_out/bench2.log
timeout 600 python bench.py > gpurun_out/bench1.log 2>&1; echo "bench1_rc=$?" >> gpurun_out/bench1.log
