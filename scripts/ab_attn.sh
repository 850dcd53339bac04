# A/B of library builds on the same box: per-kernel ncu times of one step for each .so given
for so in "$@"; do
  for rep in 1 2; do
    SV_LIBSV=$PWD/$so ncu --metrics gpu__time_duration.sum --clock-control none -s 171 -c 14 --csv --log-file gpurun_out/ab.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
    python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/ab.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print('$so', [(r[ki][:10], int(r[vi])//100/10) for r in rows[1:] if 'attn' in r[ki] or 'gemm' in r[ki]])"
  done
done
