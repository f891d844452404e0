# final-state evidence at the bench's launch shape (angle batch of 8): launch list + ncu --set full of one step's passes
set -x
mkdir -p gpurun_out
CMD="python bench.py --angles 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/fin_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 3000 --csv --log-file gpurun_out/fin_launches.csv $CMD > gpurun_out/fin_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_x1|k_y1|k_x2|k_y2|k_x3" -s 56 -c 14 -o gpurun_out/fin_prof $CMD > gpurun_out/fin_ncu2.log 2>&1
tail -2 gpurun_out/fin_ncu2.log
# post-process on the box (the report itself exceeds the 64 MiB copy-back limit)
python tools/ncu_summary.py gpurun_out/fin_prof.ncu-rep > gpurun_out/fin_summary.md 2>&1
python tools/ncu_stalls.py gpurun_out/fin_prof.ncu-rep > gpurun_out/fin_stalls.txt 2>&1
python tools/traffic_json.py gpurun_out/fin_prof.ncu-rep gpurun_out/fin_traffic.json > gpurun_out/fin_traffic.log 2>&1
ncu -i gpurun_out/fin_prof.ncu-rep --page raw --csv > gpurun_out/fin_raw.csv 2>/dev/null
python tools/launch_summary.py gpurun_out/fin_launches.csv > gpurun_out/fin_launches_summary.txt 2>&1
rm -f gpurun_out/fin_prof.ncu-rep
