#!/bin/bash
# full-size ncu captures of big_gram_tc_kernel: a user-side (launch 3) and an item-side (launch 30) batch
# usage: tools/prof_tc.sh TAG [extra tuning for tc_full_prof.py, e.g. tc_debug=2]
set -e
tag=${1:-tc}
shift || true
python tools/tc_full_prof.py large 1 "$@" > gpurun_out/${tag}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:big_gram_tc -s 3 -c 1 -o gpurun_out/${tag}_user python tools/tc_full_prof.py large 1 "$@" > gpurun_out/${tag}_ncu_u.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:big_gram_tc -s 30 -c 1 -o gpurun_out/${tag}_item python tools/tc_full_prof.py large 1 "$@" > gpurun_out/${tag}_ncu_i.log 2>&1
