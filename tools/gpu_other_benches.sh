# the other workloads' benches at the final state (compute-sanitizer is closed on this GPU pool: a first version
# of this script ran memcheck / racecheck / synccheck over the cfg0-size tests and every run was refused, exit 86)
# usage (via gpurun): bash tools/gpu_other_benches.sh [tag]
TAG=${1:-r02_san}
mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg4.log 2>&1; tail -c 1500 gpurun_out/${TAG}_bench_cfg4.log
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg2.log 2>&1; tail -c 600 gpurun_out/${TAG}_bench_cfg2.log
timeout 600 python bench.py --angles 64 --probe-shifts 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_ps.log 2>&1; tail -c 600 gpurun_out/${TAG}_bench_ps.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.log 2>&1; tail -c 800 gpurun_out/${TAG}_bench_reference.log
