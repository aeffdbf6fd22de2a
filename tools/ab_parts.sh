#!/usr/bin/env bash
# A/B of the tile list's token-order parts per expert segment (kTileParts): W reloads vs L2 reuse
for tp in 8 4 2 16; do
  MHL_NVCC_DEFS="-DMHL_TILE_PARTS=$tp" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('parts=$tp', round(d['ms_per_step'],3), 'F5', b['F5_expert_fwd'], 'K1', b['B5_expert_bwd_dx'], 'K2', b['B5_expert_dx_gemm'], 'F4', b['F4_cluster'])"
  done
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
