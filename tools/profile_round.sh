#!/bin/bash
# Round profile on a B200 (B200_PROFILING.md): (1) the plain command first, (2) the ncu launch list
# (gpu__time_duration, --clock-control none, cold-cache serialised) of 300 bench windows, (3) one
# ncu --set full capture of the three window kernels of steady-state window 181 of the C5
# workload.  Output: gpurun_out/prof/ ; then `python tools/prof_summary.py r02` writes profiles/r02/.
set -e
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --profile-run --steps 1 --warmup 0 --windows 300 --no-extra"
$CMD > $OUT/bench_plain.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
python tools/ncu_window.py --windows 182 > $OUT/window_plain.txt
ncu --set full --clock-control none --import-source on -k regex:"k_begin_coord|k_advance|k_ledger" -s 540 -c 3 \
    -o $OUT/full -f python tools/ncu_window.py --windows 182 > $OUT/ncu_full.log 2>&1
ncu -i $OUT/full.ncu-rep --page raw --csv > $OUT/full_raw.csv 2>/dev/null
ncu -i $OUT/full.ncu-rep --page details --csv > $OUT/full_details.csv 2>/dev/null
ncu -i $OUT/full.ncu-rep --page source --csv --print-source cuda,sass > $OUT/full_src.csv 2>/dev/null || true
echo done
