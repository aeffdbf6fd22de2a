#!/usr/bin/env bash
# A/B of the expert kernels' output-tile store path (LSU default vs MHL_STORE_TMA=1), then GPU tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 0 1 0 1; do
  MHL_STORE_TMA=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('tma=$v', round(d['ms_per_step'],3), 'F5', b['F5_expert_fwd'], 'K1', b['B5_expert_bwd_dx'], 'K2', b['B5_expert_dx_gemm'], 'dW', b['B5_expert_bwd_dw'])"
done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
