#!/bin/bash
# GPU-box session script (run via gpurun): tests, smoke, FP32 peak probe,
# the full bench line, the ncu launch list and one --set full capture of the
# dominant kernel (each ncu run after its command exited 0 without ncu).
# Usage: tools/gpu_round.sh [tag] [stages...]   stages: env tests smoke fp32 bench launches full
set -u
TAG=${1:-run}; shift || true
STAGES=${*:-env tests smoke fp32 bench launches full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
has() { [[ " $STAGES " == *" $1 "* ]]; }
if has env; then
  { nvidia-smi; free -g; nproc; python -c "import torch; print(torch.__version__)"; } > $OUT/env.txt 2>&1
fi
if has tests; then
  timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?" | tee -a $OUT/rc.txt
fi
if has smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
  echo "smoke rc=$?" | tee -a $OUT/rc.txt
fi
if has fp32; then
  timeout 120 ./tools/fp32_tput > $OUT/fp32_tput.txt 2>&1
  echo "fp32 rc=$?" | tee -a $OUT/rc.txt
fi
if has bench; then
  timeout 1500 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
  echo "bench rc=$?" | tee -a $OUT/rc.txt
fi
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
if has launches; then
  timeout 900 $CMD > $OUT/plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
  echo "launch list rc=$?" | tee -a $OUT/rc.txt
fi
if has full; then
  timeout 900 $CMD > $OUT/plain2.log 2>&1 && \
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"frame_cl|frame_tma|frame_rmw" -s 3 -c 1 \
      -o $OUT/prof_full $CMD > $OUT/ncu_full.log 2>&1
  echo "full capture rc=$?" | tee -a $OUT/rc.txt
fi
