timeout 600 python -m pytest tests/test_gpu_joints.py tests/test_gpu_scene.py -q > gpurun_out/r2e_joints_scene.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pile_parity.py -q > gpurun_out/r2e_pile_parity.log 2>&1
