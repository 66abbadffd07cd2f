# late-window diagnostics: Cholesky trace over [150,200) and a CUPTI timeline of step 190
ABD_TRACE_CHOL=1 timeout 600 python bench.py --no-e2e --no-full-run --no-cpu --steps 50 --warmup 3 > gpurun_out/r2_trace_bench.json 2> gpurun_out/r2_trace_chol.log
python tools/chol_trace_summary.py gpurun_out/r2_trace_chol.log 320 > gpurun_out/r2_chol_summary.txt 2>&1
timeout 600 python tools/gpu_timeline.py 1 pile bench_data/pile_step190.npz > gpurun_out/r2_timeline_step190.txt 2>&1
timeout 600 python tools/gpu_timeline.py 1 pile bench_data/pile_step150.npz > gpurun_out/r2_timeline_step150.txt 2>&1
