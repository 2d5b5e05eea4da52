#!/bin/bash
# A/B of kernel-variant builds of libptg.so on the GPU box (run via gpurun):
#   tools/ab_variants.sh TAG name1 name2 ...   ("default" = the shipped library)
# Per variant: the RMW parity tests, then bench.py --no-extras (config 5).
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for v in "$@"; do
  if [ "$v" = default ]; then unset PTG_LIB; else export PTG_LIB=$PWD/paper_1810_05628_b200/lib/variants/libptg_$v.so; fi
  timeout 900 python -m pytest tests/test_gpu_large.py -m gpu -q -x -p no:cacheprovider -k "rmw or config5 or config4_full" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$?" | tee -a $OUT/rc.txt
  for rep in 1 2; do
    timeout 600 python bench.py --no-extras --steps 10 --warmup 3 > $OUT/bench_${v}_$rep.json 2> $OUT/bench_${v}_$rep.err
    python - <<P | tee -a $OUT/rc.txt
import json
try:
    d = json.load(open("$OUT/bench_${v}_$rep.json"))
    print("$v rep $rep: %.3f ms/eval, e2e %.3f ms" % (d["ms_per_step"], d["e2e"]["ms_per_step"]))
except Exception as e:
    print("$v rep $rep: failed", e)
P
  done
done
