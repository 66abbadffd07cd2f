#!/bin/bash
# One gpurun call that produces the round's evidence under gpurun_out/ (copy the
# summaries into profiles/ afterwards):
#   /usr/local/graft/bin/gpurun --timeout 4200 -- 'bash tools/gpu_round_profile.sh TAG'
# GPU tests + smoke, the driver's bench command, DRAM traffic + FP64 flops per kernel
# group (tools/measure_traffic.py), the ncu launch list of one late step, ncu --set full
# captures of the top kernels, config 2, the other configs, 2 slab ranks on the pile.
TAG=${1:-final}
O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
ONE="python bench.py --steps 1 --warmup 0 --window-steps 1 --no-e2e --no-cpu --no-full-run"
timeout 1800 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "rc $?" >> $O/${TAG}_pytest_gpu.log
timeout 120 python __graft_entry__.py > $O/${TAG}_smoke.log 2>&1; echo "rc $?" >> $O/${TAG}_smoke.log
# the traffic capture first: it writes profiles/traffic_pile.json, which the bench line reads
timeout 1200 python tools/measure_traffic.py --workload pile --steps 1 > $O/${TAG}_measure_traffic.log 2>&1
cp profiles/fp64_peak.json $O/fp64_peak.json 2>/dev/null
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench_line.json 2> $O/${TAG}_bench.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launch_list.csv $ONE > $O/${TAG}_ncu_launch.log 2>&1
for k in k_chol_flow k_prim_pairs2 k_ccd_hot k_energy_all; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"^${k}$" -s 20 -c 1 -o $O/${TAG}_${k} $ONE > $O/${TAG}_ncu_${k}.log 2>&1
done
timeout 1500 python bench.py --workload micro --steps 3 --warmup 1 > $O/${TAG}_bench_micro.json 2> $O/${TAG}_bench_micro.err
for wl in boxstack cubes chainmail; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --start 3 --no-cpu > $O/${TAG}_bench_${wl}.json 2> $O/${TAG}_bench_${wl}.err
done
timeout 900 python tools/slab_pile.py 2 1 > $O/${TAG}_slab_pile.txt 2>&1
