mkdir -p gpurun_out/r02k
for c in 2 4; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-extras"
  timeout 600 $CMD > gpurun_out/r02k/plain$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"frame_tma|frame_cl|overlap_gather|plane_reduce" -s 4 -c 2 -o gpurun_out/r02k/prof_c$c $CMD > gpurun_out/r02k/ncu$c.log 2>&1
  echo "c$c rc=$?"
done
