mkdir -p gpurun_out/r02h
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02h/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r02h/bench.json 2> gpurun_out/r02h/bench.err; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/r02h/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['step_breakdown']['frame_kernel_ms'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --no-extras --steps 10 --config 4 > gpurun_out/r02h/bench4.json 2> gpurun_out/r02h/bench4.err; echo bench4=$?
python -c "import json;d=json.loads(open('gpurun_out/r02h/bench4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['step_breakdown']['frame_kernel_ms'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --no-extras --steps 10 --config 3 > gpurun_out/r02h/bench3.json 2> gpurun_out/r02h/bench3.err; echo bench3=$?
python -c "import json;d=json.loads(open('gpurun_out/r02h/bench3.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['step_breakdown']['frame_kernel_ms'], d['e2e']['ms_per_step'])"
