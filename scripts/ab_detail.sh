# A/B of library builds with per-stage live times: alternating `bench.py --detail` runs per .so.
# Usage: WL=ns bash scripts/ab_detail.sh a.so b.so   (prints value, ms/step, SM clock and per-stage us)
for rep in 1 2; do
  for so in "$@"; do
    SV_LIBSV=$PWD/$so timeout 300 python bench.py --workload ${WL:-ns} --steps ${STEPS:-200} --warmup 10 --e2e-steps 0 \
      --no-cpu-baseline --steady-s 0 --check-steps 0 --detail 2>/dev/null | python scripts/ab_line.py "$so"
  done
done
