#!/bin/bash
# N=1 launch list of the bench command (after the same command exits 0 without ncu)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy"
timeout 600 $CMD > gpurun_out/nl_plain.json 2> gpurun_out/nl_plain.err; echo "plain rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_n1_bench_launches.csv \
  $CMD > gpurun_out/nl_ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/r02_n1_bench_launches.csv")) if len(r) > 10]
hdr = rows[0]; ik = hdr.index("Kernel Name"); iv = hdr.index("Metric Value"); iu = hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ik].split("(")[0][:60]
    v = float(r[iv].replace(",", "")) * (1e-3 if r[iu] == "nsecond" else 1.0 if r[iu] == "usecond" else 1e3)
    c, t = agg.get(k, (0, 0.0)); agg[k] = (c + 1, t + v)
for k, (c, t) in agg.items(): print(f"{k:60s} {c:5d} {t:10.1f} us {t / c:8.2f}")
PY
