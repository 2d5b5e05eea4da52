mkdir -p gpurun_out/r02s
res() { python -c "import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],2))"; }
timeout 600 python bench.py --no-extras --steps 5 > gpurun_out/r02s/b.json 2> gpurun_out/r02s/b.err; echo "base $(res gpurun_out/r02s/b.json)"
PTG_LIB=paper_1810_05628_b200/lib/variants/libptg_bulk.so timeout 600 python bench.py --no-extras --steps 5 > gpurun_out/r02s/b.json 2> gpurun_out/r02s/b.err; echo "bulk $(res gpurun_out/r02s/b.json)"
PTG_LIB=paper_1810_05628_b200/lib/variants/libptg_bulk.so timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider -k "rmw or config5" > gpurun_out/r02s/pytest.log 2>&1; echo pytest_bulk=$?
