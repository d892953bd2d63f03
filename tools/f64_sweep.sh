# Float64 accumulation in the tiled Gram (CALS_GRAM_F64=1) vs the float64 folds: time and later-iteration accuracy.
for g in 1 0; do
  echo "== CALS_GRAM_F64=$g"
  CALS_GRAM_F64=$g timeout 600 python bench.py --no-cpu --no-e2e --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms/iter', round(d['ms_per_step'],1), {k: round(v['ms']/6,1) for k,v in d['kernels'].items() if v['ms'] > 60})"
  for w in 5 9; do CALS_GRAM_F64=$g timeout 900 python tools/ill_diag.py large $w 2>&1 | grep ratio; done
done
