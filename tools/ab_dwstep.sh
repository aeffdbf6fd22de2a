# dW A/B (under gpurun): pipeline step 32 rows x 4 stages (default) vs 64 x 2 and 16 x 8
for st in ${STLIST:-32 64 16}; do
  MHL_NVCC_DEFS="-DMHL_DW_STEP=$st" python -m paper_2602_04870_b200.build --force > /dev/null 2>&1
  echo "dw_step=$st"
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "expert_tcgen05 or paper_head or edge or weight_gradients or det" 2>&1 | tail -1
  for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], 'dW', b['B5_expert_bwd_dw'])"; done
done
