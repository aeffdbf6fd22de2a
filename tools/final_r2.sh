#!/usr/bin/env bash
# Round-2 final evidence (under gpurun): paper bench line with e2e + CPU baseline, BASELINE config
# lines, reference arm, ncu launch list + --set full of the hot kernels, compute-sanitizer passes.
TAG=${1:-r2z}
OUT=gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/${TAG}_smoke.log | cut -c1-150)"
timeout 300 python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench_paper.json 2> $OUT/${TAG}_bench_paper.err; echo "paper rc=$?"
for c in small g2x paper_k2 paper_k4 paper_k16 table5 paper_rtok; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err; echo "$c rc=$?"
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${TAG}_bench_reference.json 2>&1; echo "reference rc=$?"
KREGEX="expert_fwd_sm100|expert_bwd_h_kernel|expert_dx_gemm|expert_dw_kernel|router_sm100_kernel|router_bwd_sm100|combine_kernel|scatter" SKIP=40 COUNT=10 timeout 900 bash tools/ncu_r2.sh $TAG > $OUT/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
for tool in ${SANITIZERS:-}; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_${tool}_smoke.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${TAG}_${tool}_smoke.log | tail -1)"
done
# the opt-in fused backward (MHL_FLAG_BWD_FUSED): a bench line, one --set full capture of its kernel,
# and memcheck / racecheck of smoke() on that path
MHL_BWD_FUSED=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/${TAG}_bench_paper_fused.json 2> $OUT/${TAG}_bench_paper_fused.err; echo "paper fused rc=$?"
MHL_BWD_FUSED=1 KREGEX=expert_bwd_fused bash tools/ncu_one.sh ${TAG}_prof_fused > /dev/null 2>&1; echo "ncu fused rc=$?"
for tool in ${SANITIZERS_FUSED:-}; do
  MHL_BWD_FUSED=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_${tool}_smoke_fused.log 2>&1
  echo "fused $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${TAG}_${tool}_smoke_fused.log | tail -1)"
done
