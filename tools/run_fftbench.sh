mkdir -p gpurun_out
for b in tools/bin/fftbench_*; do echo "== $b"; timeout 120 $b; done > gpurun_out/fftbench.log 2>&1
cat gpurun_out/fftbench.log
