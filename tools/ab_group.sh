#!/usr/bin/env bash
# A/B of kTileGroup (consecutive tiles per persistent-CTA work unit)
for g in 8 4 16; do
  MHL_NVCC_DEFS="-DMHL_TILE_GROUP=$g" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('group=$g', round(d['ms_per_step'],3), 'F5', b['F5_expert_fwd'], 'K1', b['B5_expert_bwd_dx'], 'K2', b['B5_expert_dx_gemm'])"
  done
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
