timeout 600 python -m pytest tests/test_gpu_joints.py tests/test_gpu_scene.py -q > gpurun_out/r2d_joints_scene.log 2>&1
for v in 0 1; do
  if [ $v = 1 ]; then export ABD_CHOL_NO_ORDER_REUSE=1; fi
  timeout 300 python bench.py --no-e2e --no-full-run --no-cpu --steps 50 --warmup 3 > gpurun_out/r2d_window_$v.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2d_window_$v.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$v', round(d['value'],3), {n:round(v['ms']/v['launches'],4) for n,v in k.items()})" >> gpurun_out/r2d_summary.txt
done
