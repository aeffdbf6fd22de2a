# K1 A/B (under gpurun): producer warps 8 (pairs per chunk, default) vs 12 (triples)
for pwv in ${PWLIST:-8 12}; do
  MHL_NVCC_DEFS="-DMHL_K1_PW=$pwv" python -m paper_2602_04870_b200.build --force > /dev/null 2>&1
  echo "k1_pw=$pwv"
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "expert_tcgen05 or paper_head or fused" 2>&1 | tail -1
  for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], 'K1', b['B5_expert_bwd_dx'])"; done
done
