#!/bin/bash
# Run on the GPU box: bench line (no extras) for configs 1-5 -> gpurun_out/configs.jsonl
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-extras >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
done
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-extras >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
python - <<'PY'
import json
for l in open("gpurun_out/configs.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"][:8], f'{d["value"]:.4g} {d["unit"]}', f'{1e3*d["ms_per_step"]:.1f} us/eval',
          f'fp32 frac {d["roofline_fp32"]["frac"]:.3f}', f'frame {1e3*d["step_breakdown"]["frame_kernel_ms"]:.1f} us')
PY
