timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/r2g_sharded.log 2>&1
timeout 600 python -m pytest tests/test_gpu_joints.py tests/test_gpu_scene.py tests/test_gpu_parity.py -q > gpurun_out/r2g_js.log 2>&1
