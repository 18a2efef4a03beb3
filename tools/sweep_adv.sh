for mb in 1 2 3 4; do
  SF_NVCC_EXTRA="-DSF_ADV_MINB=$mb" python -m paper_2601_12784_b200.build --force > /dev/null
  echo -n "adv_minb=$mb "; python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,1), round(d['ms_per_step'],4), {k: round(v,3) for k,v in r['step_share'].items()})"
done
