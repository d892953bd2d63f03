# Parameter sweep of the 500M config under env overrides (CALS_ITEM_ROWS, CALS_CALIB_M, CALS_CALIB_Z, CALS_SMALL_KB); results go to gpurun_out/.
run() { tag=$1; shift; env $tag timeout 600 python bench.py "$@" --no-cpu --no-e2e --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$tag $*', round(d['ms_per_step'],2), {n:round(v['ms']/6,1) for n,v in k.items() if v['ms']>30})" >> gpurun_out/sweep.log; }
for kb in 150 100 190 215; do run CALS_SMALL_KB=$kb; done
