# Coordinator register budget sweep: per-route sub-step cycles (timing build) and bench (normal build).
for mb in ${MINBS:-5 4 3}; do
  SF_NVCC_EXTRA="-DSF_TIMING -DSF_TIMING_ROUTE -DSF_COORD_MINB=$mb" python -m paper_2601_12784_b200.build --force > /dev/null
  echo "minb=$mb route steps:"; python tools/route_steps.py 2>&1 | sed -n 2,4p
  SF_NVCC_EXTRA="-DSF_COORD_MINB=$mb" python -m paper_2601_12784_b200.build --force > /dev/null
  echo -n "minb=$mb bench "; python bench.py --profile-run --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,1), round(d['ms_per_step'],4), round(r['ms_per_launch'],4), {k: round(v,3) for k,v in r['step_share'].items()})"
done
