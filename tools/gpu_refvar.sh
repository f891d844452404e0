TAG=${1:-refvar}
mkdir -p gpurun_out
for lib in paper_2407_20304_b200/libholo.so build_variants/*.so; do
  echo "== $lib"
  HOLO_LIB=$lib timeout 600 python -m pytest -q -m gpu tests/test_gpu_ref.py -x 2>&1 | tail -1
  HOLO_LIB=$lib timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value %.1f frame-it/s  ms/step %.1f' % (d['value'], d['ms_per_step']))"
done > gpurun_out/${TAG}.log 2>&1
cat gpurun_out/${TAG}.log
