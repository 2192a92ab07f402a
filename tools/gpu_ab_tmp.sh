timeout 900 python -m pytest tests/test_gpu_pack.py tests/test_gpu_parity.py -x -q -k "pack or host" > gpurun_out/pt_pack.log 2>&1; tail -3 gpurun_out/pt_pack.log
for a in "--fmt u8" "--fmt u8 --no-pack-u8" "--config 2 --fmt u8" "--config 2 --fmt u8 --no-pack-u8"; do
  timeout 600 python bench.py $a --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$a', round(d['value'],1), round(d['ms_per_step'],3), d['gpu_launches'], d['e2e']['value'] if d.get('e2e') else None, d['parity']['mismatches'], d['config']['fmt'])
"
done
