python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 0 32 4 0 32; do
  MHL_DX_DBG=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print('dbg=$v', round(d['ms_per_step'],3), 'K1', b['B5_expert_bwd_dx'], 'dW', b['B5_expert_bwd_dw'], 'K2', b['B5_expert_dx_gemm'])"
done
MHL_DX_DBG=32 timeout 600 python -m pytest tests -q -m gpu -x -k "expert or paper or loopback or pair or host" 2>&1 | tail -2
