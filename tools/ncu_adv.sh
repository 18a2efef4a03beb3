# ncu source-level capture of one k_advance launch (window ~7 of the C5 bench).
python bench.py --profile-run --steps 10 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_advance --launch-skip ${SKIP:-7} --launch-count 1 \
  -o gpurun_out/adv -f python bench.py --profile-run --steps 10 > gpurun_out/ncu_adv.log 2>&1
ncu -i gpurun_out/adv.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/adv_src.csv 2>/dev/null
ncu -i gpurun_out/adv.ncu-rep --page details --csv > gpurun_out/adv_details.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/adv_src.csv 40 > gpurun_out/adv_lines.txt
tail -2 gpurun_out/ncu_adv.log
