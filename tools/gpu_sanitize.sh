# compute-sanitizer over the small-size GPU tests (cfg0: 128^2 torus, all passes incl. the staged
# copies, CG step, probe-shift path, reference arm), then the other workloads' benches at the final state
# usage (via gpurun): bash tools/gpu_sanitize.sh [tag]
TAG=${1:-r02_san}
mkdir -p gpurun_out
SEL="tests/test_gpu_parity.py::test_cfg0_gradient_parity tests/test_gpu_parity.py::test_cfg0_adjoint_parity tests/test_gpu_parity.py::test_cfg0_forward_parity tests/test_gpu_cg.py::test_cg_two_iterations_cfg0_vs_oracle tests/test_gpu_ref.py::test_ref_arm_pow2_parity_vs_c_oracle"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
    python -m pytest $SEL -x -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/${TAG}_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/${TAG}_${tool}.log | tail -3 | tee -a gpurun_out/${TAG}_summary.txt
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 --print-limit 20 \
  python -m pytest "tests/test_gpu_probe_shift.py::test_fused_cg_iteration_vs_oracle" "tests/test_gpu_parity.py::test_angle_batch_ragged_parity" -x -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_memcheck2.log 2>&1
echo "memcheck2 exit $?" | tee -a gpurun_out/${TAG}_summary.txt
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/${TAG}_memcheck2.log | tail -3 | tee -a gpurun_out/${TAG}_summary.txt
timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg4.log 2>&1; tail -c 1500 gpurun_out/${TAG}_bench_cfg4.log
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg2.log 2>&1; tail -c 600 gpurun_out/${TAG}_bench_cfg2.log
timeout 600 python bench.py --angles 64 --probe-shifts 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_ps.log 2>&1; tail -c 600 gpurun_out/${TAG}_bench_ps.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.log 2>&1; tail -c 800 gpurun_out/${TAG}_bench_reference.log
