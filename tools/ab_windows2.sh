#!/usr/bin/env bash
# windowed combine: with / without the L2 discard, and window widths (MHL_NVCC_DEFS=-DMHL_TILE_PARTS=..)
run() { timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graph "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']
print(round(d['ms_per_step'],3), {k: b.get(k) for k in ('F5_expert_fwd','F6_combine','B5_expert_dx_gemm','B6_combine_bwd')})"; }
echo -n "win+discard "; MHL_WINDOWS=1 run
echo -n "win nodisc  "; MHL_WINDOWS=1 MHL_WIN_DISCARD=0 run
echo -n "default     "; run
