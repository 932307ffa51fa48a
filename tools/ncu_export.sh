#!/bin/bash
# ncu_export.sh <report-base>: text exports of gpurun_out/<base>.ncu-rep (raw metrics CSV, details page,
# source page with SASS), then drops the report itself if it is larger than 12 MB (gpurun copies at
# most 64 MiB back).
NCU=/usr/local/cuda/bin/ncu
R=gpurun_out/$1.ncu-rep
[ -f "$R" ] || { echo "no report $R"; exit 1; }
$NCU -i "$R" --page raw --csv > gpurun_out/$1.raw.csv 2>/dev/null
$NCU -i "$R" --page details > gpurun_out/$1.details.txt 2>/dev/null
$NCU -i "$R" --page source --csv --print-source sass > gpurun_out/$1.source.csv 2>/dev/null
gzip -f gpurun_out/$1.source.csv
sz=$(stat -c %s "$R")
if [ "$sz" -gt 12000000 ]; then rm -f "$R"; echo "$1: report $sz bytes dropped after export"; fi
