mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
./scripts/micro/mix_rates > /dev/null 2>&1; true  > gpurun_out/mix_rates.jsonl 2>&1; cat gpurun_out/mix_rates.jsonl
timeout 1500 python bench.py --workload layer --steps 8 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err
echo "layer rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_layer.json').read().strip().splitlines()[-1]);print(d['value'], d['decode_ms_per_token'], d['first_token_ms'], d['prefill_ms'], d['clocks'])"
