mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 1200 python -m pytest tests/test_gpu_masks.py tests/test_gpu_hotpath.py tests/test_layer.py tests/test_snapshot.py -q -x 2>&1 | tail -2
for e in "CGB_WS_GIB=3" "CGB_WS_GIB=6" "CGB_WS_GIB=10"; do
env $e timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$e', round(d['value'],2), round(d['e2e']['value'],2), d['step_ms'], {k:v['ms'] for k,v in list(d['units'].items())[:3]})"
done
timeout 900 python bench.py --workload prefill --steps 1 --no-cpu-baseline > gpurun_out/pf.json 2> gpurun_out/pf.err; echo "prefill rc=$?"; tail -3 gpurun_out/pf.err; python -c "import json;d=json.loads(open('gpurun_out/pf.json').read().strip().splitlines()[-1]);print('prefill', d['value'], d['e2e']['value'], {k:v['ms'] for k,v in list(d['units'].items())[:4]})"
timeout 1200 python bench.py --workload layer --steps 6 --no-cpu-baseline > gpurun_out/ly.json 2> gpurun_out/ly.err; echo "layer rc=$?"; tail -3 gpurun_out/ly.err; python -c "import json;d=json.loads(open('gpurun_out/ly.json').read().strip().splitlines()[-1]);print('layer', d['value'], d['decode_ms_per_token'], d['first_token_ms'], d['prefill_ms'], {k:v['ms'] for k,v in list(d['units'].items())[:6]})"
