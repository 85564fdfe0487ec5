#!/bin/bash
O=gpurun_out/g4; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none --csv --log-file $O/l13b_m2.csv python tools/fwd_one.py opt-1.3b 1 2 2 2 > $O/l13b_m2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none --csv --log-file $O/l13b_m256.csv python tools/fwd_one.py opt-1.3b 32 8 2 3 > $O/l13b_m256.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/l13_m256.csv python tools/fwd_one.py opt-13b 32 8 2 3 > $O/l13_m256.log 2>&1
