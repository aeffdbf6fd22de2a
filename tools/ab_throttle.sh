#!/usr/bin/env bash
# K1: ring depth x global progress throttle (MHL_K1_RING6, MHL_K1_THROTTLE)
for defs in "" "-DMHL_K1_THROTTLE" "-DMHL_K1_RING6 -DMHL_K1_THROTTLE"; do
  MHL_NVCC_DEFS="$defs" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
    timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('[$defs]', round(d['ms_per_step'],3), 'K1', b['B5_expert_bwd_dx'])"
  done
  MHL_NVCC_DEFS="$defs" timeout 300 python -m pytest tests -q -x -m gpu -k "expert or paper or loopback" 2>&1 | tail -1
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
