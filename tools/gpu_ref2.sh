TAG=${1:-ref2}
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_ref.py tests/test_gpu_init.py -k "ref or probe" -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg4.log 2>&1
python - gpurun_out/${TAG}_bench_cfg4.log <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
d=json.loads(l[-1]); print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), d['roofline'])
PY
CMD="python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
