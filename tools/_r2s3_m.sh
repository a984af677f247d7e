mkdir -p gpurun_out
timeout 600 python tools/a7_check.py --net inception_v3 > gpurun_out/s3m_a7_inception.log 2>&1; tail -2 gpurun_out/s3m_a7_inception.log
timeout 600 python tools/a7_check.py --net squeezenet > gpurun_out/s3m_a7_squeezenet.log 2>&1; tail -2 gpurun_out/s3m_a7_squeezenet.log
timeout 900 python tools/merge_probe.py --batch 32 --stages "8,9,11;17,18,20;97,98,101;99,100;103,104" > gpurun_out/s3m_merge_b32.log 2>&1; tail -8 gpurun_out/s3m_merge_b32.log
