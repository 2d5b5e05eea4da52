#!/bin/bash
# Run on the GPU box (via gpurun): full bench line, then the ncu launch list and
# one --set full capture of the dominant kernel, each after the identical
# command has exited 0 without ncu.  Outputs land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
echo "bench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-extras"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
$CMD > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"frame_tma|overlap_gather|plane_reduce" -s 6 -c 2 \
    -o $OUT/prof_full $CMD > $OUT/ncu_full.log 2>&1
echo "full capture rc=$?"
