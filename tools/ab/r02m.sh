mkdir -p gpurun_out/r02m
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider -k "rmw or config5" > gpurun_out/r02m/pytest.log 2>&1; echo pytest=$?
PTG_LIB=paper_1810_05628_b200/lib/variants/libptg_tl.so python tools/rmw_timeline.py 5 > gpurun_out/r02m/tl5.txt 2>&1
timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r02m/bench.json 2> gpurun_out/r02m/bench.err; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/r02m/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['step_breakdown']['frame_kernel_ms'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
