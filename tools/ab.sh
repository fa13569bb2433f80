# A/B: alternate the in-tree build and ab/*.so on the same box (bench.py C2, no e2e / CPU arm)
run() { python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["stages_ms"]["multicrop"])'; }
for r in 1 2; do
  echo "tree $(run)"
  for f in ab/*.so; do echo "$(basename $f) $(PF_B200_LIB=$PWD/$f run)"; done
done
