mkdir -p gpurun_out/r02o
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"frame_rmw2" -s 2 -c 1 -o gpurun_out/r02o/prof_rmw2 $CMD > gpurun_out/r02o/ncu.log 2>&1; echo ncu=$?
