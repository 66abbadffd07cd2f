ABD_CHOL_DUMP_GRAPH=gpurun_out/graph190.bin timeout 600 python tools/gpu_timeline.py 1 pile bench_data/pile_step190.npz > /dev/null 2>&1
./tools/ubench/chol_order_bench gpurun_out/graph190.bin > gpurun_out/chol_order_bench_box.txt 2>&1
nproc >> gpurun_out/chol_order_bench_box.txt; lscpu | head -20 >> gpurun_out/chol_order_bench_box.txt
./tools/ubench/dfma > gpurun_out/fp64_peak.json 2> gpurun_out/dfma.err
timeout 1200 python tools/measure_traffic.py --workload pile --steps 1 > gpurun_out/measure_traffic_pile.log 2>&1
