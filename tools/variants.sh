# time tuning-variant builds of libholo (HOLO_LIB) on a short cfg3 bench; parity of each on cfg0/cfg1
mkdir -p gpurun_out
ANG=${ANG:-16}
for lib in paper_2407_20304_b200/libholo.so ${VARIANTS:-build_variants/*.so}; do
  echo "== $lib"
  HOLO_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cfg0 or cfg1 or torus" 2>&1 | tail -1
  HOLO_LIB=$lib timeout 600 python bench.py --angles $ANG --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value %.1f frame-it/s  ms/step %.1f' % (d['value'], d['ms_per_step']))
for k,v in d['passes'].items(): print('   %-7s %8.2f ms/step  %6.1f GB/s  %5.1f TF' % (k, v['ms_per_step'], v['GBps'], v['TFLOPs']))
"
done > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
