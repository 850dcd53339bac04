# A/B of library builds on one box: ncu per-kernel serial times of one ns step, then alternating
# short live benches (CUDA events) per .so. Usage: bash scripts/ab_live.sh a.so b.so
for so in "$@"; do
  SV_LIBSV=$PWD/$so ncu --metrics gpu__time_duration.sum --clock-control none -s 171 -c 14 --csv --log-file gpurun_out/ab_$(basename $so).csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/ab_$(basename $so).csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print('$so ncu', [(r[ki][:8], int(r[vi])//100/10) for r in rows[1:] if 'attn' in r[ki]])"
done
for rep in 1 2; do
  for so in "$@"; do
    SV_LIBSV=$PWD/$so timeout 300 python bench.py --steps ${STEPS:-200} --warmup 10 --e2e-steps 0 --no-cpu-baseline --steady-s 0 --check-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernels']; print('$so live', d['value'], d['ms_per_step'], k['attention']['us_per_launch'], k['attention']['frac'], d['clocks']['sm_mhz'])"
  done
done
