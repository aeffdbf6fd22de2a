#!/usr/bin/env bash
# ncu evidence at HEAD (under gpurun): launch list of bench steps + one --set full capture of every
# hot kernel of the paper-scale step.  Numbers printed under ncu are never bench values.
TAG=${1:-r2}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $B > /dev/null 2>&1; echo "launches rc=$?"
python tools/ncu_summary.py launches $OUT/${TAG}_launches.csv > $OUT/${TAG}_launches.txt 2>&1; head -30 $OUT/${TAG}_launches.txt
K=${KREGEX:-"expert_fwd_sm100|expert_bwd_h_kernel|expert_dx_gemm|expert_dw_kernel|router_sm100_kernel|router_bwd_sm100|combine_kernel|scatter|tile_prefix"}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-40} -c ${COUNT:-11} -o $OUT/${TAG}_prof python bench.py --steps 1 --warmup 4 --no-e2e --no-cpu-baseline > $OUT/${TAG}_prof.log 2>&1; echo "prof rc=$?"
tail -3 $OUT/${TAG}_prof.log
