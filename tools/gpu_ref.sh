# one GPU call: engine CTA-split microbenchmark, new parity tests, cfg4 bench + ncu of the reference-arm kernels
TAG=${1:-ref}
mkdir -p gpurun_out
for b in tools/bin/fftbench*; do echo "== $b"; timeout 120 $b; done > gpurun_out/${TAG}_fftbench.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_ref.py tests/test_gpu_multires.py -k "tau or object_only or probe_subset" > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg4.log 2>&1; tail -c 1500 gpurun_out/${TAG}_bench_cfg4.log
CMD="python bench.py --workload cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ref" -s 40 -c 6 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
