# F3 A/B (under gpurun): epilogue warpgroups of the router (3 default, 4)
for eg in ${EGLIST:-3 4}; do
  MHL_NVCC_DEFS="-DMHL_ROUTER_EG=$eg" python -m paper_2602_04870_b200.build --force > /dev/null 2>&1
  echo "router_eg=$eg"
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "router or k_sweep_paper or edge" 2>&1 | tail -1
  for r in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], 'F3', b['F3_router_topk'])"; done
done
