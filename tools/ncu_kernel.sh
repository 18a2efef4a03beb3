# ncu source-level capture of one launch of a window kernel: KERNEL=<regex> SKIP=<launches to skip>
K=${KERNEL:-k_ledger}
python bench.py --profile-run --steps 10 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip ${SKIP:-7} --launch-count 1 \
  -o gpurun_out/kern -f python bench.py --profile-run --steps 10 > gpurun_out/ncu_kern.log 2>&1
ncu -i gpurun_out/kern.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/kern_src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/kern_src.csv 30 > gpurun_out/kern_lines.txt
tail -2 gpurun_out/ncu_kern.log
