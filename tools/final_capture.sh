# Round-end evidence: bench lines (ours + reference arm), launch list and full captures of the top kernel.
set -x
python bench.py > gpurun_out/f_bench_large.log 2>&1
python bench.py --impl reference > gpurun_out/f_bench_reference_large.log 2>&1
python bench.py --config medium > gpurun_out/f_bench_medium.log 2>&1
python bench.py --config powerlaw > gpurun_out/f_bench_powerlaw.log 2>&1
ncu --kernel-name-base demangled -k regex:cals:: --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/f_large_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/f_ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:big_gram -c 1 -o gpurun_out/f_user_big_gram \
    python tools/prof_half.py large user 1 > gpurun_out/f_ncu_user.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "target/" -k regex:big_gram -c 1 \
    -o gpurun_out/f_item_big_gram python tools/prof_half.py large item 1 > gpurun_out/f_ncu_item.log 2>&1
