# in-situ A/B of wgrad tile variants (LPP_WGRAD_VARIANT per C = 16, 32, 64)
F="--steps 200 --warmup 10 --no-cpu --no-sweep --no-rn18 --no-rn50 --no-baselines --no-bf16 --no-e2e"
for v in ${VARIANTS:-"0,0,0" "0,0,2" "0,0,3" "0,0,0" "0,0,2"}; do
  LPP_WGRAD_VARIANT=$v python bench.py $F 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']))"
done
