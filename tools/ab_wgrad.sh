#!/usr/bin/env bash
# dW_out GEMM overlapped with the B6 combine (side stream) vs inside B8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 0 1 0 1; do
  MHL_OVERLAP_WGRAD=$v timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('overlap=$v', round(d['ms_per_step'],3), 'B8', b['B8_proj_out_bwd'], 'B6', b['B6_combine_bwd'], 'B1', b['B1_proj_in_bwd'])"
done
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -1
