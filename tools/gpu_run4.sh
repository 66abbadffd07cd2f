timeout 300 python bench.py --no-e2e --no-full-run --no-cpu --steps 50 --warmup 3 > gpurun_out/r2b_window.json 2>/dev/null
python -c "import json,sys; d=json.loads(open('gpurun_out/r2b_window.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print(round(d['value'],3), {n:round(v['ms']/v['launches'],4) for n,v in k.items()})" > gpurun_out/r2b_summary.txt
timeout 600 python tools/gpu_timeline.py 1 pile bench_data/pile_step190.npz > gpurun_out/r2b_timeline_step190.txt 2>&1
ABD_TRACE_CHOL=1 timeout 600 python tools/gpu_timeline.py 1 pile bench_data/pile_step190.npz > /dev/null 2> gpurun_out/r2b_trace190.log
