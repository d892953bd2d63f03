# round-end measurement batch (run on the GPU box from the repo root): GPU tests, smoke, the bench lines of
# every config and the reference arm, the ncu launch list and one --set full capture of the dominant kernel
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/r02_bench_large.json 2> gpurun_out/bench_large.err; echo large rc=$?
for c in small medium powerlaw; do python bench.py --config $c > gpurun_out/r02_bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; done
python bench.py --impl reference > gpurun_out/r02_bench_reference_large.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
python bench.py --config wide --no-e2e --no-cpu > gpurun_out/r02_bench_wide.json 2> gpurun_out/bench_wide.err; echo wide rc=$?
K='regex:^(big_|small_gram|tiny_gram|solve_|refine_|quantile_table|tc_scales|sum_partial|finish_sum|residual|sqnorm|fast_)'
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 1200 --csv --log-file gpurun_out/r02_large_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo ncu rc=$?
ncu --set full --import-source on --clock-control none -k regex:big_gram_tc -s 16 -c 1 -f -o gpurun_out/r02_tc_final python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_tc.log 2>&1; echo ncu2 rc=$?
