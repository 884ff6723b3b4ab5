#!/bin/bash
# Sample SM clock / power / throttle reasons while a command runs:  tools/power_probe.sh CMD...
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,temperature.gpu,clocks_throttle_reasons.sw_power_cap,clocks_throttle_reasons.hw_slowdown --format=csv,noheader -lms 250 > /tmp/pp.csv &
P=$!
"$@"
kill $P
sort /tmp/pp.csv | uniq -c | sort -k1 -nr | head -12
