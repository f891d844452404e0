TAG=${1:-ref3}
mkdir -p gpurun_out
CMD="python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_ref_r1b|k_ref_r3b|k_ref_r2b" -s 64 -c 3 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
