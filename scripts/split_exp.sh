for k in 1024 2048 4096; do
  if [ $k = 1024 ]; then unset SV_LIBSV; else export SV_LIBSV=$PWD/gpurun_exp_libsv_$k.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -s 171 -c 14 --csv --log-file gpurun_out/sp_$k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/sp_$k.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print('split $k', [(r[ki][:10], int(r[vi])//1000) for r in rows[1:] if 'attn' in r[ki]])"
done
