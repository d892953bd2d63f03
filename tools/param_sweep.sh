# Parameter sweep under env overrides (CALS_ITEM_ROWS, CALS_CALIB_M, CALS_CALIB_Z, CALS_ILL_RATIO); results in gpurun_out/.
run() { tag=$1; shift; env $tag timeout 600 python bench.py "$@" --no-cpu --no-e2e --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); k=d['kernels']; print('$tag $*', round(d['ms_per_step'],2), {n:round(v['ms']/6,1) for n,v in k.items() if v['ms']>30})" >> gpurun_out/sweep.log; }
for r in 100 30 10; do run CALS_ILL_RATIO=$r; done
