#!/bin/bash
# Round-end measurement on one B200 (gpurun): smoke, the GPU suite, complete-run bench lines of every
# config (default launch), the reference arm, then the ncu round profile (tools/profile_round.sh).
# Output in gpurun_out/; copied into profiles/<round>/ by hand.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_multirank.py > gpurun_out/gputests.txt 2>&1
echo rc=$? >> gpurun_out/gputests.txt
for c in C1 C2 C3; do python bench.py --workload $c --steps 3 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python bench.py --workload C4 --steps 1 --warmup 3 --cpu-seconds 30 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/profile_round.sh > gpurun_out/prof_round.log 2>&1
