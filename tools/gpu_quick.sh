#!/bin/bash
# quick GPU check of a kernel change: short pile bench (device pass only), then the
# candidate-set / pile parity / exactness tests
#   gpurun --timeout 1500 -- 'bash tools/gpu_quick.sh TAG'
T=${1:-q}
timeout 400 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-full-run > gpurun_out/${T}_b.json 2> gpurun_out/${T}_b.err
timeout 900 python -m pytest tests/test_gpu_pile_parity.py tests/test_gpu_exact_opts.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${T}_t.log 2>&1; echo rc $? >> gpurun_out/${T}_t.log
