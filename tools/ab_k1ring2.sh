#!/usr/bin/env bash
# K1 ring depth (4 / 6 stages) x gather L2 policy (evict_last default / evict_normal: MHL_DX_DBG=16)
for defs in "" "-DMHL_K1_RING6"; do
  MHL_NVCC_DEFS="$defs" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for dbg in 0 16; do
    MHL_DX_DBG=$dbg timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('[$defs] dbg=$dbg', round(d['ms_per_step'],3), 'K1', b['B5_expert_bwd_dx'])"
  done
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
