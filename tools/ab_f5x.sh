# F5 A/B (under gpurun, timing only: xdbg != 0 gives wrong results): X gathers of random rows (0),
# the same gather4 stream over consecutive rows (1), no gathers (2)
for d in 0 1 2; do
  echo "xdbg=$d"
  MHL_F5_XDBG=$d timeout 300 python bench.py --config small --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('small', d['ms_per_step'])" 
  MHL_F5_XDBG=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('paper F5', d['step_breakdown_ms']['F5_expert_fwd'])"
done
