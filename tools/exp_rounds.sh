run() { python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["stages_ms"], d["sampler"])'; }
for r in 4 2 1 4 2 1; do echo "rounds=$r $(PF_SAMPLER_ROUNDS=$r run)"; done
