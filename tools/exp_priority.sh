run() { python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["stages_ms"]["multicrop"], d["stages_ms"]["sample_wait"])'; }
for p in -1 0; do
  echo "prio=$p tree $(PF_SAMPLER_PRIORITY=$p run)"
  for f in ab/*.so; do echo "prio=$p $(basename $f) $(PF_SAMPLER_PRIORITY=$p PF_B200_LIB=$PWD/$f run)"; done
done
