#!/usr/bin/env bash
# IMAD / IMAD.HI / IMAD.WIDE issue rates (tools/imad_microbench.cu) with the SM clock and
# throttle reasons sampled by nvidia-smi while it runs (the clock record of the peak).
#   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/imad_mb.bin tools/imad_microbench.cu
#   tools/run_imad_mb.sh > profiles/rN_imad_microbench.txt
set -euo pipefail
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw \
  --format=csv,noheader -lms 20 > /tmp/imad_clk.csv &
smi=$!
sleep 0.3
for i in 1 2 3; do ./tools/imad_mb.bin; done
kill $smi
echo "# nvidia-smi samples during the runs (timestamp, sm MHz, max MHz, reasons, power):"
sort -t, -k2 /tmp/imad_clk.csv | awk -F, '{print $2}' | sort | uniq -c
tail -3 /tmp/imad_clk.csv
