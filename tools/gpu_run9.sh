./tools/ubench/dfma > gpurun_out/fp64_peak.json 2> gpurun_out/dfma.err
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/r2f_sharded.log 2>&1
timeout 600 python -m pytest tests/test_gpu_joints.py tests/test_gpu_scene.py tests/test_gpu_pile_parity.py -q > gpurun_out/r2f_js.log 2>&1
timeout 300 python - > gpurun_out/r2f_boxits.txt 2>&1 <<'P'
import warnings, numpy as np, sys
sys.path.insert(0, 'tests')
import paper_2201_10022_b200 as P
from test_gpu_parity import _box_stack_model
g = np.load('tests/golden/box_stack.npz')
model, state, params = _box_stack_model(g)
its = []
warnings.simplefilter('ignore')
for s in range(len(g['iterations'])):
    state, st = P.advance_step(model, state, params)
    its.append(st.iterations)
d = [(k, a, int(b)) for k, (a, b) in enumerate(zip(its, g['iterations'])) if a != b]
print('box stack iteration mismatches', d, sum(its), int(g['iterations'].sum()))
P
