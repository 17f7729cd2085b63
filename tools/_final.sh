timeout 600 python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final2_ref.json 2> gpurun_out/final2_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/final2_ncu_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'dstE|thomas' --csv --log-file gpurun_out/final2_solve_launches.csv python tools/one_solve.py --cfg 4 --reps 3 > gpurun_out/final2_ncu_solve.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'dstE|thomas' -s 5 -c 5 -o gpurun_out/final2_full python tools/one_solve.py --reps 2 > gpurun_out/final2_ncu_full.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final2_gputest.log 2>&1; tail -2 gpurun_out/final2_gputest.log
