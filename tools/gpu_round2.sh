# Round-2 measurement pass on one B200: smoke, GPU tests, bench (+ reference arm),
# ncu launch list of the headline step, one ncu --set full capture of every
# composite component (-> profiles traffic), SASS is extracted on the CPU side.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:randomly > gpurun_out/pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest.log
fi
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref_rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown --no-c5 > gpurun_out/bench_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"scan_lag|scan_smem|mapreduce_kernel|gevm_cols|gemv_kernel|code_sum" -o /tmp/comp python tools/ncu_components.py run > gpurun_out/ncu_comp.log 2>&1
ncu -i /tmp/comp.ncu-rep --page raw --csv > gpurun_out/comp_raw.csv 2>/dev/null
ncu -i /tmp/comp.ncu-rep --page details --csv > gpurun_out/comp_details.csv 2>/dev/null
python tools/ncu_components.py summarize gpurun_out/comp_raw.csv gpurun_out/r02_summary > gpurun_out/ncu_summary.log 2>&1
ls -la gpurun_out
