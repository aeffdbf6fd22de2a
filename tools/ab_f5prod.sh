# F5 A/B (under gpurun): 8 producer warps in pairs + 4 Y warps (default) vs 4 whole-chunk producer warps + 8 Y warps
OUT=gpurun_out
for pwv in ${PWLIST:-8 4}; do
  MHL_NVCC_DEFS="-DMHL_F5_PROD_WARPS=$pwv" python -m paper_2602_04870_b200.build --force > /dev/null 2>&1
  echo "prod_warps=$pwv"
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "expert_tcgen05 or paper_head or small_bf16" 2>&1 | tail -1
  MHL_TRACE_FWD=$OUT/f5p$pwv.trace timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python tools/trace_fwd.py $OUT/f5p$pwv.trace | grep -E "period\(20\)|10->20|23->24|21->22"
  for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], 'F5', b['F5_expert_fwd'])"; done
  timeout 300 python bench.py --config small --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('small', d['ms_per_step'])"
done
