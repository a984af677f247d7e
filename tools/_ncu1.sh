mkdir -p gpurun_out
python bench.py --steps 30 --warmup 5 --cpu-sample-s 1 --save-schedule gpurun_out/r2_sched_inc2.json > gpurun_out/r2_bench2.log 2>&1; tail -1 gpurun_out/r2_bench2.log | cut -c1-400
ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2_ncu_launches.csv python tools/ncu_run.py --schedule gpurun_out/r2_sched_inc2.json > gpurun_out/r2_ncu_run.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -s 8 -c 4 -f -o gpurun_out/r2_stage_full python tools/ncu_run.py --schedule gpurun_out/r2_sched_inc2.json > gpurun_out/r2_ncu_full.log 2>&1
tail -2 gpurun_out/r2_ncu_full.log; ls -la gpurun_out/
