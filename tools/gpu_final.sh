# round-end evidence in one GPU call: smoke, the full -m gpu suite, the default bench,
# then the launch list + one ncu --set full capture of the passes at the bench's launch shape
# usage (via gpurun): bash tools/gpu_final.sh [tag]
TAG=${1:-r02_end}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
( time python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/${TAG}_smoke.log 2>&1; tail -3 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -15 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; tail -c 3000 gpurun_out/${TAG}_bench.log
CMD="python bench.py --angles 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 3000 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_x1|k_y1|k_x2|k_y2|k_x3" -s 20 -c 16 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
tail -2 gpurun_out/${TAG}_ncu2.log
python tools/ncu_summary.py gpurun_out/${TAG}_prof.ncu-rep > gpurun_out/${TAG}_summary.md 2>&1
python tools/ncu_stalls.py gpurun_out/${TAG}_prof.ncu-rep > gpurun_out/${TAG}_stalls.txt 2>&1
python tools/traffic_json.py gpurun_out/${TAG}_prof.ncu-rep gpurun_out/${TAG}_traffic.json > gpurun_out/${TAG}_traffic.log 2>&1
rm -f gpurun_out/${TAG}_prof.ncu-rep
ls -la gpurun_out | tail -20
