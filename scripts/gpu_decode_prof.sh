#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/decode64_launches.csv python scripts/decode_launches.py 64 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/decode64_launches.csv > gpurun_out/decode64_summary.txt 2>&1
timeout 300 python scripts/decode_profile.py > gpurun_out/decode_profile.txt 2>&1
