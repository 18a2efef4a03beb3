for mb in 5 6 7 8; do
  SF_NVCC_EXTRA="-DSF_COORD_MINB=$mb" python -m paper_2601_12784_b200.build --force > /dev/null
  echo -n "minb=$mb "; python bench.py --profile-run --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,1), round(d['ms_per_step'],4), {k: round(v,3) for k,v in r['step_share'].items()})"
done
