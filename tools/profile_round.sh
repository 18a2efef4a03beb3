#!/bin/bash
# Round profile of the C5 bench command: the ncu launch list (gpu__time_duration, cold-cache,
# serialised) and one ncu --set full capture of the three window kernels at window 60.
# The same command first runs without ncu (B200_PROFILING.md).  Output: gpurun_out/prof/.
set -e
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --profile-run --steps 3 --warmup 60"
$CMD > $OUT/bench_plain.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_begin_coord|k_advance|k_ledger" -s 180 -c 3 \
    -o $OUT/full -f $CMD > $OUT/ncu_full.log 2>&1
ncu -i $OUT/full.ncu-rep --page raw --csv > $OUT/full_raw.csv 2>/dev/null
ncu -i $OUT/full.ncu-rep --page details --csv > $OUT/full_details.csv 2>/dev/null
ncu -i $OUT/full.ncu-rep --page source --csv --print-source cuda,sass > $OUT/full_src.csv 2>/dev/null || true
echo done
