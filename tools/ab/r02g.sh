mkdir -p gpurun_out/r02g
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_large.py -m gpu -q -p no:cacheprovider > gpurun_out/r02g/pytest.log 2>&1; echo pytest=$?
python -c "
import time, numpy as np
from paper_1810_05628_b200 import Plan, synth
cfg = synth.CONFIGS[5]
obj, probe, pos = synth.make_inputs(cfg)
t = time.time(); p = Plan(cfg.n, cfg.M, cfg.w, pos, None, probe, precision='c64'); print('plan create s', time.time() - t)
" > gpurun_out/r02g/create.log 2>&1
timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r02g/bench.json 2> gpurun_out/r02g/bench.err; echo bench=$?
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/r02g/memcheck.log 2>&1; echo memcheck=$?
