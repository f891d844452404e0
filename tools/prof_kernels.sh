# ncu --set full of the line kernels on a short bench (4 angles); usage: bash tools/prof_kernels.sh "<regex>" <skip> <count>
set -x
mkdir -p gpurun_out
RE=${1:-"k_y2|k_x2"}
SKIP=${2:-100}
CNT=${3:-4}
CMD="python bench.py --angles 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT -o gpurun_out/prof $CMD > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
