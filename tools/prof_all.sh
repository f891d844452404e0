# bench + launch list + ncu --set full of the five line passes (one GPU)
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1
CMD="python bench.py --angles 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 3000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_x1|k_y1|k_x2|k_y2|k_x3" -s 60 -c 5 -o gpurun_out/prof $CMD > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
ls -la gpurun_out; du -sh gpurun_out
