# F5 A/B (under gpurun): Y staging stages (MHL_F5_YSTAGES; 1 -> a 5-stage X ring), F5 span + trace
OUT=gpurun_out
for ys in ${YSLIST:-2 1}; do
  MHL_NVCC_DEFS="-DMHL_F5_YSTAGES=$ys" python -m paper_2602_04870_b200.build --force > /dev/null 2>&1
  MHL_TRACE_FWD=$OUT/f5ys$ys.trace timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "ystages=$ys"; python tools/trace_fwd.py $OUT/f5ys$ys.trace | grep -E "period|10->20|23->24"
  for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], b['F5_expert_fwd'])"; done
  MHL_F5_XDBG=2 timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no-gather F5', d['step_breakdown_ms']['F5_expert_fwd'])"
done
