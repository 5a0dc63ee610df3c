LOPT_TRACE=1 python -m paper_2506_10315_b200.build --force > /dev/null 2>&1
LOPT_APPLY_DEBUG=32 timeout 200 python tools/trace_apply.py > gpurun_out/trace_$1.txt 2>&1; tail -3 gpurun_out/trace_$1.txt
