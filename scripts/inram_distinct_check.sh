timeout 600 python -m pytest tests/test_gpu_ring_host.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --ring host_batch --distinct --sweep 128,1024,4096 --steps 1000 --warmup 50 --no-e2e --no-gather --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l); print(d['config']['batch'], round(d['value']))
    except: pass"
