#!/usr/bin/env bash
# One --set full capture (with source) of the first launch matching KREGEX in a bench step
# (under gpurun).  Usage: KREGEX=... [ENVS] bash tools/ncu_one.sh TAG
TAG=$1
OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${SKIP:-0} -c 1 \
  -o $OUT/${TAG} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${BENCHARGS} > $OUT/${TAG}.log 2>&1
echo "ncu $TAG rc=$?"; tail -2 $OUT/${TAG}.log
