for c in 1 1.5 2 3 4 6; do
  ABD_CHOL_LOOKAHEAD=$c timeout 300 python bench.py --no-e2e --no-full-run --no-cpu --steps 50 --warmup 3 > gpurun_out/la_$c.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/la_$c.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$c', round(d['value'],3), {n:round(v['ms']/v['launches'],4) for n,v in k.items()})" >> gpurun_out/la_summary.txt
done
