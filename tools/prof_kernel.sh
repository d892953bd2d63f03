#!/bin/bash
# full-size ncu capture of one launch of a kernel during one iteration of the large config
# usage: tools/prof_kernel.sh TAG KERNEL_REGEX LAUNCH_SKIP [tuning k=v ...]
set -e
tag=$1; kre=$2; skip=$3
shift 3
python tools/tc_full_prof.py large 1 "$@" > gpurun_out/${tag}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${kre} -s ${skip} -c 1 -o gpurun_out/${tag} python tools/tc_full_prof.py large 1 "$@" > gpurun_out/${tag}_ncu.log 2>&1
