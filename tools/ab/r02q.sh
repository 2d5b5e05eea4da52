mkdir -p gpurun_out/r02q
res() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],2))"; }
for v in "PTG_RMW_PAIR=0" "PTG_RMW_PAIR=6" "PTG_RMW_PAIR=7"; do
  env $v timeout 600 python bench.py --no-extras --steps 5 > gpurun_out/r02q/b.json 2> gpurun_out/r02q/b.err; echo "c5 $v $(res gpurun_out/r02q/b.json)"
done
for v in "PTG_RMW=1 PTG_RMW_PAIR=0" "PTG_RMW=1 PTG_RMW_PAIR=4" "PTG_RMW=0"; do
  env $v timeout 600 python bench.py --config 4 --no-extras --steps 5 > gpurun_out/r02q/b.json 2> gpurun_out/r02q/b.err; echo "c4 $v $(res gpurun_out/r02q/b.json)"
done
timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider -k "rmw" > gpurun_out/r02q/pytest.log 2>&1; echo pytest=$?
