# Alternating live benches of two library builds on ns, c2 and c3 (attention + step time).
for rep in 1 2; do for so in gpurun_exp_base.so gpurun_exp_chain.so; do for w in ns c2 c3; do
SV_LIBSV=$PWD/$so timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernels']; print('$so $w', d['value'], d['ms_per_step'], k['attention']['us_per_launch'], k['attention']['frac'], d['clocks']['sm_mhz'])"
done; done; done
