#!/bin/bash
# ncu --set full capture of one kernel, exported to CSV pages on the GPU box
# (a full report with source counters can exceed gpurun's 64 MiB return limit).
# usage: tools/ncu_capture.sh <name> <kernel-regex> <skip> -- <command...>
set -u
name=$1; regex=$2; skip=$3; shift 4
ncu -f --set full --import-source on --clock-control none -k "regex:$regex" -s "$skip" -c 1 \
    -o "/tmp/$name" "$@" > "gpurun_out/$name.log" 2>&1
for page in details raw source; do
  ncu -i "/tmp/$name.ncu-rep" --page $page --csv > "gpurun_out/${name}_$page.csv" 2>/dev/null
done
gzip -f gpurun_out/${name}_source.csv gpurun_out/${name}_raw.csv
ls -la gpurun_out | tail -5
