# Timing of the routing decision: per-route sub-step cycles (SF_TIMING_ROUTE build), then bench.
for v in ${VARIANTS:-""}; do
  SF_NVCC_EXTRA="-DSF_TIMING -DSF_TIMING_ROUTE -DSF_COORD_MINB=4 $v" python -m paper_2601_12784_b200.build --force > /dev/null
  echo "variant [$v]:"; python tools/route_steps.py 2>&1 | sed -n 2,3p
done
SF_NVCC_EXTRA="-DSF_COORD_MINB=4" python -m paper_2601_12784_b200.build --force > /dev/null
echo -n "bench "; python bench.py --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,1), round(d['ms_per_step'],4), round(r['ms_per_launch'],4), {k: round(v,3) for k,v in r['step_share'].items()})"
