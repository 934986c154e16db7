# Quick GPU pass (development): smoke, scan/mapreduce probes, tests, bench, 2-rank bench path.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/probe.py scan > gpurun_out/probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:randomly > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
FORGE_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --elems 268435456 > gpurun_out/bench2.log 2>&1; echo "bench2_rc=$?" >> gpurun_out/bench2.log
