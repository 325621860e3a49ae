mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --workload layer --steps 8 > gpurun_out/bench_layer.json 2> gpurun_out/bench_layer.err
echo "layer rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_layer.json').read().strip().splitlines()[-1]);print(d['value'], d['decode_ms_per_token'], d['first_token_ms'], d['prefill_ms'], d['clocks'], d['cpu_baseline']['value'])"
timeout 600 python scripts/host_profile.py > gpurun_out/host_profile.txt 2>&1; head -45 gpurun_out/host_profile.txt
cd baseline/_ref/cryptogen_tests && PYTHONPATH=/root/repo/baseline/_ref:/root/repo:/root/repo/tests CGB_KEY_SEED=0 timeout 1500 python -m pytest -q -p ref_dropin_plugin -p no:cacheprovider --rootdir . -o addopts= test_model.py test_acceptance.py test_costmodel.py --durations=10 > /root/repo/gpurun_out/ref_suite_more.log 2>&1; echo "more rc=$?"; tail -20 /root/repo/gpurun_out/ref_suite_more.log
