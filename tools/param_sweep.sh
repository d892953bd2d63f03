# Parameter sweep of the 500M config under env overrides (CALS_ITEM_ROWS, CALS_CALIB_M, CALS_CALIB_Z); results go to gpurun_out/.
run() { tag=$1; shift; env $tag timeout 600 python bench.py "$@" --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$tag $*', round(d['ms_per_step'],3))" >> gpurun_out/v18_sweep.log; }
for c in medium powerlaw; do
run CALS_ITEM_ROWS=4096 --config $c
run X=0 --config $c
done
