mkdir -p gpurun_out
for B in 4 8 16; do
  timeout 600 python bench.py --angles 32 --batch $B --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --multires-angles 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$B value %.1f frame-it/s  ms/step %.1f' % (d['value'], d['ms_per_step']))
for k,v in d['passes'].items(): print('   %-7s %8.2f ms/step  %8.1f us/frame' % (k, v['ms_per_step'], v.get('us_per_frame', 0)))
"
done > gpurun_out/batch.log 2>&1
cat gpurun_out/batch.log
