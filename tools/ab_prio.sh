# A/B of stream priorities (MGB_STREAM_PRIORITY=1) against the default: bench value, e2e, config 1
mkdir -p gpurun_out/prio
for v in 1 0 1 0; do
  MGB_STREAM_PRIORITY=$v timeout 300 python bench.py --songs 0 --no-cpu-baseline --no-secondary > gpurun_out/prio/b_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/prio/b_$v.json').read().strip().splitlines()[-1]); print('prio=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['config1']['value'],1))" >> gpurun_out/prio/ab.txt
done
