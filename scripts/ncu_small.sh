# Per-kernel memory / occupancy metrics of one timed ns step (serialised ncu replay): duration, DRAM
# bytes, L2 hit rate, achieved occupancy. Usage: SO=path/libsv.so bash scripts/ncu_small.sh tag
tag=${1:-small}
SV_LIBSV=$PWD/${SO:-paper_2604_09562_b200/libsv.so} ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size \
  --clock-control none -s 171 -c 14 --csv --log-file gpurun_out/ncu_${tag}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --steady-s 0 --check-steps 0 > /dev/null 2>&1
python - "$tag" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/ncu_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
k = collections.OrderedDict()
for r in rows[1:]:
    k.setdefault((r[ii], r[ki][:28]), {})[r[mi]] = r[vi]
for (i, n), m in k.items():
    print(f"{n:28s} us {float(m['gpu__time_duration.sum'].replace(',',''))/1e3:7.1f} rdMB {float(m['dram__bytes_read.sum'].replace(',',''))/1e6:8.1f} "
          f"wrMB {float(m['dram__bytes_write.sum'].replace(',',''))/1e6:7.1f} L2hit {m['lts__t_sector_hit_rate.pct']:>6s} "
          f"occ {m['sm__warps_active.avg.pct_of_peak_sustained_active']:>6s} regs {m['launch__registers_per_thread']} grid {m['launch__grid_size']}")
PY
