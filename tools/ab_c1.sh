# config-1 throughput by sampler prefetch chunk (PF_REGION_CHUNK; default 1024 // batch)
run() { python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["stages_ms"])'; }
for c in 4 8 16 32; do echo "chunk=$c $(PF_REGION_CHUNK=$c run)"; done
