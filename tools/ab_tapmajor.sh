# the forward weight staging: tap-major copy per call (C >= 32, default) vs per-CTA transpose
F="--steps 200 --warmup 10 --no-cpu --no-sweep --no-rn18 --no-rn50 --no-baselines --no-bf16 --no-e2e"
for m in 32 1000 32 1000; do
  LPP_CONV_TAPMAJOR_MIN_C=$m python bench.py $F 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('min_c $m', round(d['value']))"
done
