QTT_ROUND_TRACE=1 python tools/c3_round.py 2 2>&1 | tail -130 > gpurun_out/trace_c3_b.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/c3_round.py 2 > /dev/null 2>&1
python tools/agg_launches.py gpurun_out/c3_launches.csv > gpurun_out/c3_launches.txt
