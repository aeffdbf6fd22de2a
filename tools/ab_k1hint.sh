#!/usr/bin/env bash
# K1 dH/gA store L2 policy: evict_first (1, default) vs normal (0)
for h in 1 0; do
  MHL_NVCC_DEFS="-DMHL_K1_STOREHINT=$h" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2 3; do
    timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('hint=$h', round(d['ms_per_step'],3), 'K1', b['B5_expert_bwd_dx'], 'K2', b['B5_expert_dx_gemm'], 'dW', b['B5_expert_bwd_dw'])"
  done
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
