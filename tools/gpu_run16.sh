for v in base nounion nounion_noreuse; do
  unset ABD_CHOL_NO_UNION ABD_CHOL_NO_ORDER_REUSE
  if [ $v = nounion ]; then export ABD_CHOL_NO_UNION=1; fi
  if [ $v = nounion_noreuse ]; then export ABD_CHOL_NO_UNION=1 ABD_CHOL_NO_ORDER_REUSE=1; fi
  timeout 300 python bench.py --no-e2e --no-full-run --no-cpu --steps 50 --warmup 3 > gpurun_out/r2j_window_$v.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2j_window_$v.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$v', round(d['value'],3), {n:round(v['ms']/v['launches'],4) for n,v in k.items()})" >> gpurun_out/r2j_summary.txt
done
