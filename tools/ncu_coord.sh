# ncu source-level capture of one heavy-window coordinator launch (window ~95 of the C5 bench).
python -m paper_2601_12784_b200.build > /dev/null
python bench.py --profile-run --steps 100 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_begin_coord --launch-skip ${SKIP:-94} --launch-count 1 \
  -o gpurun_out/coord_heavy -f python bench.py --profile-run --steps 100 > gpurun_out/ncu_coord.log 2>&1
ncu -i gpurun_out/coord_heavy.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/coord_heavy_src.csv 2>/dev/null
ncu -i gpurun_out/coord_heavy.ncu-rep --page details --csv > gpurun_out/coord_heavy_details.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/coord_heavy_src.csv 45 > gpurun_out/coord_heavy_lines.txt
tail -3 gpurun_out/ncu_coord.log
