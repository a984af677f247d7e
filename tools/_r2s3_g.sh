mkdir -p gpurun_out
export IOS_LIB=paper_2011_01302_b200/build/libios_fine.so IOS_TRACE_FINE_NAMES=1
python tools/trace_stage.py inception_v3 "[([5],0),([56,60,63],0),([53,54,57],0),([97,99,100,103,104,106],0),([120],0)]" > gpurun_out/s3g_trace_fine.log 2>&1
unset IOS_LIB IOS_TRACE_FINE_NAMES
timeout 3600 python bench.py --net nasnet_a_large --steps 50 --warmup 5 --cpu-sample-s 5 --latency-cache gpurun_out/f4_lc_nasnet.txt --save-schedule gpurun_out/f4_sched_nasnet_a_large.json > gpurun_out/f4_bench_nasnet_a_large.log 2>&1
tail -1 gpurun_out/f4_bench_nasnet_a_large.log | cut -c1-300
du -sh gpurun_out
