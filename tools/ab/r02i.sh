mkdir -p gpurun_out/r02i
res() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['step_breakdown']['frame_kernel_ms'],3), round(d['e2e']['ms_per_step'],2))"; }
for sb in 1024 512 1536 32; do
  PTG_RMW_SB=$sb timeout 600 python bench.py --no-extras --steps 8 > gpurun_out/r02i/b.json 2> gpurun_out/r02i/b.err; echo "c5 sb=$sb $(res gpurun_out/r02i/b.json)"
done
for v in "PTG_RMW=0" "PTG_RMW=1"; do
  env $v timeout 600 python bench.py --no-extras --steps 8 --config 4 > gpurun_out/r02i/b.json 2> gpurun_out/r02i/b.err; echo "c4 $v $(res gpurun_out/r02i/b.json)"
done
timeout 600 python bench.py --no-extras --steps 8 --config 3 > gpurun_out/r02i/b.json 2> gpurun_out/r02i/b.err; echo "c3 $(res gpurun_out/r02i/b.json)"
