#!/bin/bash
# Full measurement pass of the current build (one box): every workload's bench line, the ns launch list,
# ncu --set full captures of the lm-head and the verify attention, the sampled finalize captures.
# Usage: bash scripts/round_measure.sh <tag>   (outputs under gpurun_out/<tag>_*)
tag=${1:-r02s3}
o=gpurun_out
python bench.py > $o/${tag}_bench_ns.json 2> $o/${tag}_bench_ns.err
for w in c2 c3 c4 ns_tree c2_filter toy; do
  python bench.py --workload $w --steps 100 > $o/${tag}_bench_$w.json 2> $o/${tag}_bench_$w.err
done
for w in ns c2 c3 toy; do
  python bench.py --workload $w --steps 100 --graph --no-cpu-baseline --e2e-steps 0 > $o/${tag}_bench_${w}_graph.json 2> $o/${tag}_bench_${w}_graph.err
done
bash scripts/profile_round.sh $tag
for w in c2 c3; do
  ncu --set full --import-source on --clock-control none -k regex:finalize_kernel -s 5 -c 1 -o $o/${tag}_fin_$w \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --steady-s 0 --check-steps 0 > /dev/null 2>&1
done
ls -la $o/${tag}_*
