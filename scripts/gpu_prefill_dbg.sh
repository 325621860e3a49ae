mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --workload prefill --steps 1 --no-cpu-baseline > gpurun_out/pf.json 2> gpurun_out/pf.err; echo "rc=$?"; tail -20 gpurun_out/pf.err; tail -c 600 gpurun_out/pf.json
for c in 0 64 128; do for rep in 1 2; do CGB_KS_CHUNK=$c timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>gpurun_out/b_$c.err | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('chunk $c', round(d['value'],2), round(d['e2e']['value'],2), d['step_ms'], {k:v['ms'] for k,v in list(d['units'].items())[:2]})"; done; done
