mkdir -p gpurun_out
python tools/stage_times.py --schedule profiles/r2_sched_inception.json > gpurun_out/s3b_stage_times.log 2>&1
python tools/trace_stage.py inception_v3 "[([1,2,3],0),([4],0),([17,18,19,20,21,22,23,24],0),([53,54,57],1),([55,58,59,62],0),([56,60,63],0),([97,99,103,104,106],0),([107],0),([96],0)]" > gpurun_out/s3b_trace.log 2>&1
