#!/bin/bash
# Profiling pass of one round, run on the GPU box from the repo root:
#   bash tools/profile_round.sh <tag>   -> gpurun_out/summary/<tag>_*.txt (ncu_summary + SASS mix per op)
# then copy gpurun_out/summary/* into profiles/ here
# (the numbers under ncu are cold-cache and serialised: never a bench value)
out=gpurun_out
mkdir -p $out
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $out/launches.csv \
    python bench.py --only drelu --steps 30 --warmup 0 > $out/ncu_launches.log 2>&1
for op in drelu relu ladder drelu_literal; do
  ncu --set full --clock-control none --import-source on -k regex:'k_fused|k_ladder' -s 2 -c 1 -f -o $out/prof_$op \
      python bench.py --only $op --steps 3 --warmup 0 > $out/ncu_$op.log 2>&1
done
# the other kernel families: every launch of one step (RSS, full precision, the party phases)
for spec in drelu_rss:1 drelu_fp:1 party_relu:5; do
  op=${spec%:*}; k=${spec#*:}   # k = launches per step; capture the second step
  ncu --set full --clock-control none --import-source on -k regex:'^k_' -s $k -c $k -f -o $out/prof_$op \
      python bench.py --only $op --steps 2 --warmup 0 > $out/ncu_$op.log 2>&1
done
# summaries on the box (the .ncu-rep files are too large to bring back in one call)
tag=${1:-r1}
python tools/ncu_summary.py $tag $out/prof_*.ncu-rep --launches $out/launches.csv --out $out/summary
for r in $out/prof_*.ncu-rep; do
  op=$(basename $r .ncu-rep); op=${op#prof_}
  python tools/sass_mix.py $r $((1<<24)) --top 30 > $out/summary/${tag}_${op}_sass_mix.txt 2>&1
done
# per-instruction source view of the headline kernel (stall samples, executed counts) for offline reading
ncu -i $out/prof_drelu.ncu-rep --page source --csv --print-source sass > $out/summary/${tag}_drelu_source.csv 2>&1
rm -f $out/prof_*.ncu-rep
ls -la $out $out/summary
