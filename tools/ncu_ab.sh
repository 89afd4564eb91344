#!/bin/bash
# Per-kernel durations at ncu's locked base clock (comparable across boxes and
# builds, unlike free-running power-capped clocks): one short bench run per
# config.  usage: tools/ncu_ab.sh TAG  -> gpurun_out/ab_TAG_<config>.csv
TAG=$1
for cfg in ${CONFIGS:-C2 C3}; do
  ncu --metrics gpu__time_duration.sum -c ${COUNT:-300} --csv --log-file gpurun_out/ab_${TAG}_${cfg}.csv \
      python bench.py --config $cfg --steps 1 --warmup 1 --no-compare --no-cpu-baseline --no-e2e \
      > gpurun_out/ab_${TAG}_${cfg}.log 2>&1
done
