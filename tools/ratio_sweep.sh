# Pivot-spread deferral ratio at n_f = 64: time per iteration and later-iteration accuracy (gpurun_out/ratio.log).
for r in 31 60 15; do
  echo "== CALS_ILL_RATIO=$r"
  CALS_ILL_RATIO=$r timeout 600 python bench.py --no-cpu --no-e2e --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms/iter', round(d['ms_per_step'],1))"
  for w in 5 9; do CALS_ILL_RATIO=$r timeout 900 python tools/ill_diag.py large $w 2>&1 | grep ratio; done
done
