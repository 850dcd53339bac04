#!/bin/bash
# Profiles for the round's commit: launch list (serialised, cold) of 4 bench steps and one
# `ncu --set full` capture each of the lm-head GEMM and the attention kernel inside a step.
# Usage: bash scripts/profile_round.sh <tag>   (outputs under gpurun_out/)
tag=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none -s 171 -c 56 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_sw_kernel -s 19 -c 1 \
    -o gpurun_out/${tag}_lm_head python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_tc2_kernel -s 3 -c 1 \
    -o gpurun_out/${tag}_attention python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la gpurun_out/${tag}_*
