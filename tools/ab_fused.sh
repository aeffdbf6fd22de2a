#!/usr/bin/env bash
# A/B of the fused (in-kernel) forward combine vs the separate combine kernel, then GPU tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_fused_small.py 2>&1 | tail -3
for v in 0 1 0 1; do
  MHL_FUSED_COMBINE=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('fused=$v', round(d['ms_per_step'],3), 'F5', b['F5_expert_fwd'], 'F6', b.get('F6_combine'))"
done
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
