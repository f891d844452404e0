# source-level stall hot spots of one kernel (regex $1), post-processed on the box
set -x
mkdir -p gpurun_out
RE=${1:-k_x3s}
CMD="python bench.py --angles 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/hx_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s 4 -c 1 -o gpurun_out/hx_prof $CMD > gpurun_out/hx_ncu.log 2>&1
python tools/ncu_hotspots.py gpurun_out/hx_prof.ncu-rep > gpurun_out/hx_hotspots_$RE.txt 2>&1
ncu -i gpurun_out/hx_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/hx_source_$RE.csv 2>/dev/null
rm -f gpurun_out/hx_prof.ncu-rep
