mkdir -p gpurun_out
for v in 0 3; do
IOS_TILE_VARIANT=$v timeout 300 python tools/stage_times.py --variants 0 --schedule profiles/r2_sched_inception.json > gpurun_out/s3e_st_v$v.log 2>&1
done
python tools/trace_stage.py inception_v3 "[([56,60,63],0)]" > gpurun_out/s3e_trace_v0.log 2>&1
IOS_TILE_VARIANT=3 IOS_DUMP_PLANS=1 python tools/trace_stage.py inception_v3 "[([56,60,63],0)]" > gpurun_out/s3e_trace_v3.log 2>&1
