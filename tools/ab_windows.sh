#!/usr/bin/env bash
# A/B of the windowed combine (MHL_WINDOWS=0: one expert launch + one combine launch)
run() { timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']
print(round(d['ms_per_step'],3), {k: b.get(k) for k in ('F5_expert_fwd','F6_combine','B5_expert_dx_gemm','B6_combine_bwd','B5_expert_bwd_dw')})"; }
for r in 1 2; do echo -n "windows "; MHL_WINDOWS=1 run; echo -n "off     "; run; done
