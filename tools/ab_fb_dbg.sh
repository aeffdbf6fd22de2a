# fused B5 A/B (under gpurun): store switches (MHL_FB_DBG 1: no dH/gA stores, 2: no dX stores, 3: none)
OUT=gpurun_out
for d in 0 1 2 3; do
  MHL_BWD_FUSED=1 MHL_FB_DBG=$d MHL_TRACE_FB=$OUT/fbdbg$d.trace timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "dbg=$d"; python tools/trace_fb.py $OUT/fbdbg$d.trace | grep -E "2->14|period\(20\)|21->22|24->25"
  MHL_BWD_FUSED=1 MHL_FB_DBG=$d timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['step_breakdown_ms']['B5_expert_bwd_dx'])"
done
