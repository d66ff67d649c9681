#!/bin/bash
# Profiling pass of one round, run on the GPU box from the repo root:
#   bash tools/profile_round.sh            -> gpurun_out/launches.csv, gpurun_out/prof_{drelu,relu,ladder}.ncu-rep
# then here: python tools/ncu_summary.py <tag> gpurun_out/prof_*.ncu-rep --launches gpurun_out/launches.csv
# (the numbers under ncu are cold-cache and serialised: never a bench value)
out=gpurun_out
mkdir -p $out
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $out/launches.csv \
    python bench.py --only drelu --steps 30 --warmup 0 > $out/ncu_launches.log 2>&1
for op in drelu relu ladder; do
  ncu --set full --clock-control none --import-source on -k regex:'k_fused|k_ladder' -s 2 -c 1 -f -o $out/prof_$op \
      python bench.py --only $op --steps 3 --warmup 0 > $out/ncu_$op.log 2>&1
done
ls -la $out
