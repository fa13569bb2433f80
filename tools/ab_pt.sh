run() { python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["stages_ms"]["read"], d["roofline"]["frac"])'; }
for r in 1 2; do echo "tree $(run)"; for f in ab/pt*.so; do echo "$(basename $f) $(PF_B200_LIB=$PWD/$f run)"; done; done
