mkdir -p gpurun_out/r02n
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02n/pytest.log 2>&1; echo pytest=$?
res() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['step_breakdown']['frame_kernel_ms'],3), round(d['e2e']['ms_per_step'],2), round(d['roofline']['frac'],4))"; }
for v in "PTG_RMW2=1" "PTG_RMW2=0"; do
  env $v timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r02n/b.json 2> gpurun_out/r02n/b.err; echo "$v $(res gpurun_out/r02n/b.json)"
done
