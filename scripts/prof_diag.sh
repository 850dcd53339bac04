for dg in 0 8 2; do
SV_SW_DIAG=$dg ncu --metrics gpu__time_duration.sum --clock-control none -s 171 -c 14 --csv --log-file gpurun_out/l_$dg.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/l_$dg.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print('diag $dg', [(int(r[vi])//1000) for r in rows[1:] if 'gemm_sw' in r[ki]])"
done
