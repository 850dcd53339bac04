# A/B of library builds on one box: ncu per-kernel times of one step + a short live bench, per .so
for so in "$@"; do
  SV_LIBSV=$PWD/$so ncu --metrics gpu__time_duration.sum --clock-control none -s 171 -c 14 --csv --log-file gpurun_out/ab.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/ab.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
v=[(r[ki][:4], int(r[vi])//100/10) for r in rows[1:]]
print('$so', v, round(sum(x[1] for x in v),1))"
  SV_LIBSV=$PWD/$so timeout 300 python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$so live', d['value'], d['ms_per_step'], d['kernels']['attention']['us_per_launch'], d['kernels']['lm_head']['us_per_launch'])"
done
