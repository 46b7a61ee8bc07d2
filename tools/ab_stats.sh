for v in acc; do cp abvar/$v.so paper_1708_08180_b200/libccl.so; timeout 300 python tools/bench_stats.py >> gpurun_out/bstats.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:k_stats --csv --log-file gpurun_out/ncu_stats.csv python tools/bench_stats.py > /dev/null 2>&1
