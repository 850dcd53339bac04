# Live (CUDA-event) per-stage times of the ns step under different conditions (one box)
B="python bench.py --e2e-steps 0 --no-cpu-baseline"
J='import json,sys; d=json.load(sys.stdin); k=d["kernels"]; print(d["ms_per_step"], d["clocks"], k["attention"]["us_per_launch"], k["lm_head"]["us_per_launch"], d.get("stages"))'
echo short60;   timeout 300 $B --steps 60 --warmup 5 2>/dev/null | python -c "$J"
echo long200;   timeout 300 $B --steps 200 --warmup 10 2>/dev/null | python -c "$J"
echo detail200; timeout 300 $B --steps 200 --warmup 10 --detail 2>/dev/null | python -c "$J"
echo nopdl200;  SV_PDL=0 timeout 300 $B --steps 200 --warmup 10 2>/dev/null | python -c "$J"
