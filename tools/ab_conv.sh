F="--steps 200 --warmup 10 --no-cpu --no-sweep --no-rn18 --no-rn50 --no-baselines"
LPP_CONV=cudnn python bench.py $F > gpurun_out/ab_cudnn.json 2> gpurun_out/ab_cudnn.err
python bench.py $F > gpurun_out/ab_native.json 2> gpurun_out/ab_native.err
python -c "
import json
for k in ('cudnn','native'):
    d=json.loads(open(f'gpurun_out/ab_{k}.json').read().strip().splitlines()[-1])
    print(k, round(d['value']), round(d['e2e']['value']), 'bf16', round(d['value_bf16']), 'frac', d['roofline']['frac'], d['ms_per_step'])
"
python -m pytest tests/test_conv_gpu.py tests/test_bench_config_gpu.py tests/test_oracle_golden.py -q -x 2>&1 | tail -3
