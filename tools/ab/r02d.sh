mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02d/pytest.log 2>&1; echo pytest=$?
for v in "PTG_RMW_BANDS=8" "PTG_RMW_BANDS=16" "PTG_RMW_BANDS=4" "PTG_NO_BANDED=1"; do
  env $v timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/r02d/bench.json'));print(d['ms_per_step'], d['step_breakdown']['frame_kernel_ms'], d['e2e']['ms_per_step'])")"
done
