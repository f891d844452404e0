# quick GPU iteration: engine microbenchmarks, parity subset, short bench
TAG=${1:-q}
mkdir -p gpurun_out
for b in tools/bin/fftbench_*; do echo "== $b"; timeout 120 $b; done > gpurun_out/${TAG}_fftbench.log 2>&1; cat gpurun_out/${TAG}_fftbench.log
timeout 900 python -m pytest tests -q -m gpu -x -k "not full_size and not cfg4" > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
python - gpurun_out/${TAG}_bench.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'binding', d['roofline_step'])
for k,v in d['passes'].items(): print('  %-7s %7.1f ms/step %8s us/frame  fp32 %.3f' % (k, v['ms_per_step'], round(v.get('us_per_frame',0),1), v['fp32_frac']))
PY
