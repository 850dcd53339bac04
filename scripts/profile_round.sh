#!/bin/bash
# Profiles for the round's commit (ns workload): the per-kernel launch list (serialised, cold) of a short
# bench run and one `ncu --set full` capture each of the lm-head GEMM and the verify attention inside a
# step. Usage: bash scripts/profile_round.sh <tag>   (outputs under gpurun_out/)
tag=${1:-r02}
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --steady-s 0 --check-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_sw_kernel -s 19 -c 1 -o gpurun_out/${tag}_lm_head $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_tc2_kernel -s 3 -c 1 -o gpurun_out/${tag}_attention $B > /dev/null 2>&1
ls -la gpurun_out/${tag}_*
