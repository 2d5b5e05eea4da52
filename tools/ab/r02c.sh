mkdir -p gpurun_out/r02c
timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02c/pytest.log 2>&1; echo pytest=$?
for v in "PTG_RMW_L=32" "PTG_RMW_L=16" "PTG_RMW_L=16 PTG_LIB=paper_1810_05628_b200/lib/variants/libptg_b4.so"; do
  env $v timeout 600 python bench.py --no-extras --steps 10 > gpurun_out/r02c/bench.json 2> gpurun_out/r02c/bench.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/r02c/bench.json'));print(d['ms_per_step'], d['step_breakdown']['frame_kernel_ms'], d['e2e']['ms_per_step'])")"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"frame_rmw" -s 2 -c 1 -o gpurun_out/r02c/prof_rmw16 python bench.py --no-extras --steps 2 --warmup 3 > gpurun_out/r02c/ncu.log 2>&1; echo ncu=$?
