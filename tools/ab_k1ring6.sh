# K1 A/B (under gpurun): the grouped epilogue stores dH/gA from registers, so its 32 KB staging can
# go to the gather ring (MHL_K1_RING6: 6 stages instead of 4)
for defs in "" "-DMHL_K1_RING6"; do
  MHL_NVCC_DEFS="$defs" python -m paper_2602_04870_b200.build --force > /dev/null 2>&1
  echo "defs=[$defs]"
  for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], 'K1', b['B5_expert_bwd_dx'])"; done
done
