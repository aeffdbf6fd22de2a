#!/usr/bin/env bash
# K1 with the default 4-stage ring vs a 6-stage ring (grouped epilogue's staging smem given to the
# ring): per-CTA duration spread (MHL_TRACE_DX, events 60/61) and bench time
for defs in "" "-DMHL_K1_RING6"; do
  MHL_NVCC_DEFS="$defs" python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('[$defs]', round(d['ms_per_step'],3), 'K1', b['B5_expert_bwd_dx'])"
  MHL_TRACE_DX=gpurun_out/trace_ring$defs.txt timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/trace_cta.py gpurun_out/trace_ring$defs.txt; python tools/trace_k1.py gpurun_out/trace_ring$defs.txt | tail -4
done
python -c "from paper_2602_04870_b200.build import build; build(force=True)" > /dev/null 2>&1
