# Float64 fold granularity of the tiled Gram: time per iteration and later-iteration accuracy (gpurun_out/fold.log).
for f in 4 8 16; do
  echo "== CALS_FOLD_CHUNKS=$f"
  CALS_FOLD_CHUNKS=$f timeout 600 python bench.py --no-cpu --no-e2e --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ms/iter', round(d['ms_per_step'],1))"
  for w in 5 9; do CALS_FOLD_CHUNKS=$f timeout 900 python tools/ill_diag.py large $w 2>&1 | grep ratio; done
done
