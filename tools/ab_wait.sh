#!/usr/bin/env bash
# A/B of the mbarrier try_wait suspend-time hint (sm100.cuh MHL_WAIT_HINT_NS), bench step breakdown.
for H in ${HINTS:-0 20000 1000000}; do
  MHL_NVCC_DEFS="-DMHL_WAIT_HINT_NS=$H" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']
print('hint=$H', round(d['ms_per_step'],3), {k: b[k] for k in ('F5_expert_fwd','B5_expert_bwd_dx','B5_expert_dx_gemm','B5_expert_bwd_dw','F3_router_topk','B3_router_bwd')})"
  done
done
