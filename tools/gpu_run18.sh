timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pile_parity.py -x -q > gpurun_out/r2l_tests.log 2>&1
for v in split nosplit; do
  unset ABD_CHOL_NO_SPLIT
  if [ $v = nosplit ]; then export ABD_CHOL_NO_SPLIT=1; fi
  timeout 300 python bench.py --no-e2e --no-full-run --no-cpu --steps 50 --warmup 3 > gpurun_out/r2l_window_$v.json 2> gpurun_out/r2l_window_$v.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2l_window_$v.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$v', round(d['value'],3), {n:round(v['ms']/v['launches'],4) for n,v in k.items()})" >> gpurun_out/r2l_summary.txt
  ABD_TRACE_CHOL=1 timeout 600 python tools/gpu_timeline.py 1 pile bench_data/pile_step190.npz > gpurun_out/r2l_timeline190_$v.txt 2> gpurun_out/r2l_trace190_$v.log
done
