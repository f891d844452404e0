TAG=${1:-fo}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fourier.py tests/test_gpu_cg.py tests/test_gpu_multires.py -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -15 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --angles 32 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --multires-angles 0 > gpurun_out/${TAG}_bench.log 2>&1
python - gpurun_out/${TAG}_bench.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'binding', d['roofline_step'])
for k,v in d['passes'].items(): print('  %-7s %7.1f ms/step %8s us/frame  fp32 %.3f' % (k, v['ms_per_step'], round(v.get('us_per_frame',0),1), v['fp32_frac']))
PY
