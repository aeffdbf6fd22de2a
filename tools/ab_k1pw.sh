#!/usr/bin/env bash
# A/B of the backward H kernel's producer-warp count (MHL_K1_PW=4|8), bench breakdown + trace
for pw in 4 8; do
  MHL_NVCC_DEFS="-DMHL_K1_PW=$pw" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('pw=$pw', round(d['ms_per_step'],3), 'K1', b['B5_expert_bwd_dx'], 'F5', b['F5_expert_fwd'])"
  done
  MHL_TRACE_DX=gpurun_out/trace_pw$pw.txt timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/trace_k1.py gpurun_out/trace_pw$pw.txt
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
