#!/usr/bin/env bash
# A/B of the GELU reciprocal split (MHL_GELU_NR: half the reciprocals by Newton steps on the FMA pipe)
for defs in "" "-DMHL_GELU_NR"; do
  MHL_NVCC_DEFS="$defs" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('[$defs]', round(d['ms_per_step'],3), 'F5', b['F5_expert_fwd'], 'K1', b['B5_expert_bwd_dx'])"
  done
  MHL_NVCC_DEFS="$defs" timeout 600 python -m pytest tests -q -x -m gpu -k "expert or paper or pair or small" 2>&1 | tail -1
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
