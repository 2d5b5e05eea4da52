mkdir -p gpurun_out/r02p
res() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],2))"; }
for v in "PTG_E2E_STREAMS=1" "PTG_E2E_STREAMS=2" "PTG_E2E_STREAMS=1 PTG_RMW_BANDS=32" "PTG_E2E_STREAMS=1 PTG_RMW_BANDS=8"; do
  env $v timeout 600 python bench.py --no-extras --steps 5 > gpurun_out/r02p/b.json 2> gpurun_out/r02p/b.err; echo "$v $(res gpurun_out/r02p/b.json)"
done
