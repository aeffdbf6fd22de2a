# F5 iteration (under gpurun): parity tests of the expert forward, CTA-0 trace, F5 span (paper, x2) and the small config
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "expert_tcgen05 or paper_head or small or k_sweep or smoke" > $OUT/f5_tests.log 2>&1; echo tests rc=$?; tail -1 $OUT/f5_tests.log
MHL_TRACE_FWD=$OUT/f5.trace timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; python tools/trace_fwd.py $OUT/f5.trace | grep -E "period|->"
for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['step_breakdown_ms']; print(d['ms_per_step'], 'F5', b['F5_expert_fwd'])"; done
timeout 300 python bench.py --config small --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('small', d['ms_per_step'])"
