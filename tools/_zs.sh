python tools/one_solve.py --cfg 4 --reps 1 --time && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'dstE|thomas' --csv --log-file gpurun_out/launches_r02.csv python tools/one_solve.py --cfg 4 --reps 1 --time > gpurun_out/ncu_l.log 2>&1
python tools/one_solve.py --cfg 4 --reps 1 --time && \
ncu --set full --clock-control none --import-source on -k regex:'thomas' -s 1 -c 1 -o gpurun_out/z_r02 python tools/one_solve.py --cfg 4 --reps 1 --time > gpurun_out/ncu_f.log 2>&1
python tools/one_solve.py --cfg 4 --reps 1 --time && \
ncu --set full --clock-control none --import-source on -k regex:'dstE' -s 9 -c 1 -o gpurun_out/ix_r02 python tools/one_solve.py --cfg 4 --reps 1 --time > gpurun_out/ncu_f2.log 2>&1
python tools/stencil_rate.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'s27_tile' -c 1 -o gpurun_out/s27_r02 python tools/stencil_rate.py > gpurun_out/ncu_s.log 2>&1
du -sh gpurun_out/*
