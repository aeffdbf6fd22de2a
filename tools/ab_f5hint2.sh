#!/usr/bin/env bash
# F5 L2 policies: 0 none, 1 gathers evict_last + stores evict_first, 2 stores evict_first only
for h in 0 2 1; do
  MHL_NVCC_DEFS="-DMHL_F5_L2HINT=$h" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2 3; do
    timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('hint=$h', round(d['ms_per_step'],3), 'F5', b['F5_expert_fwd'], 'F6', b['F6_combine'])"
  done
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
