#!/usr/bin/env bash
# A/B: default kernels vs CTA-pair expert kernels (MHL_FLAG_PAIR) vs pair K1 with the single-CTA F5
run() { timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']
print(round(d['ms_per_step'],3), {k: b[k] for k in ('F5_expert_fwd','B5_expert_bwd_dx','B5_expert_dx_gemm','B5_expert_bwd_dw','F6_combine','B6_combine_bwd')})"; }
for r in 1 2; do echo -n "default "; run; echo -n "pair    "; run --pair; echo -n "pairK1  "; MHL_F5_SINGLE=1 run --pair; done
