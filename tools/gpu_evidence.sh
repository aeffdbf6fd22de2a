#!/usr/bin/env bash
# One GPU pass producing the round's evidence (run under gpurun from the repo root):
#   GPU parity tests, smoke, the bench JSON line, the ncu launch list of a bench step and
#   one `ncu --set full` capture of the dominant kernels.  Output under gpurun_out/<tag>_*.
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -q -m gpu > $OUT/${TAG}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/${TAG}_gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
tail -1 $OUT/${TAG}_bench.json | cut -c1-400
# launch list of one timed step (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
for k in ${NCU_KERNELS:-expert_bwd_h expert_dw_kernel expert_fwd_sm100 expert_dx_gemm combine_bwd}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o $OUT/${TAG}_prof_$k \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu $k rc=$?"
done
