# time tuning-variant builds of libholo (HOLO_LIB) on a short cfg3 bench, with a parity subset per variant
mkdir -p gpurun_out
ANG=${ANG:-16}
TAG=${TAG:-v}
for lib in paper_2407_20304_b200/libholo.so ${VARIANTS:-build_variants/*.so}; do
  echo "== $lib"
  HOLO_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg.py -x -q -m gpu -k "not full_size" 2>&1 | tail -1
  HOLO_LIB=$lib timeout 150 python bench.py --angles $ANG --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value %.1f frame-it/s  ms/step %.1f' % (d['value'], d['ms_per_step']))
for k,v in d['passes'].items(): print('   %-7s %8.2f ms/step  %8.1f us/frame  %5.1f TF' % (k, v['ms_per_step'], v.get('us_per_frame', 0), v['TFLOPs']))
"
done > gpurun_out/${TAG}_variants.log 2>&1
cat gpurun_out/${TAG}_variants.log
