set -x
export PYTHONUNBUFFERED=1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy"
timeout 600 $CMD > gpurun_out/n1_plain.json 2> gpurun_out/n1_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n1_launches.csv $CMD > gpurun_out/n1_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_flat_tma -s 3 -c 1 -o gpurun_out/n1_full -f $CMD > gpurun_out/n1_ncu2.log 2>&1
timeout 300 python tools/prof_pack.py > gpurun_out/pack.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pack|k_unpack" -s 2 -c 2 -o gpurun_out/pack_full -f python tools/prof_pack.py > gpurun_out/pack_ncu.log 2>&1
echo done
