# full validation + bench + profiles (round 2, r2i)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2i_pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/r2i_pytest_gpu.log
timeout 120 python __graft_entry__.py > gpurun_out/r2i_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2i_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2i_bench_line.json 2> gpurun_out/r2i_bench.err
timeout 900 python tools/slab_pile.py 2 1 > gpurun_out/r2i_slab_pile.txt 2>&1
timeout 1200 python tools/measure_traffic.py --workload pile --steps 1 > gpurun_out/r2i_measure_traffic.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launch_list.csv python bench.py --steps 1 --warmup 0 --window-steps 1 --no-e2e --no-cpu --no-full-run > gpurun_out/r2i_ncu_launch.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_chol_sched -s 20 -c 1 -o gpurun_out/r2i_chol python bench.py --steps 1 --warmup 0 --window-steps 1 --no-e2e --no-cpu --no-full-run > gpurun_out/r2i_ncu_chol.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_prim_pairs2 -s 20 -c 1 -o gpurun_out/r2i_prim python bench.py --steps 1 --warmup 0 --window-steps 1 --no-e2e --no-cpu --no-full-run > gpurun_out/r2i_ncu_prim.log 2>&1
