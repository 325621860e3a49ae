mkdir -p gpurun_out
python -c "import paper_2602_08798_b200._native as n; n.build()" > gpurun_out/build.log 2>&1
make -s -C oracle
timeout 600 python -m pytest tests/test_gpu_threads.py -q 2>&1 | tail -2
cd baseline/_ref/cryptogen_tests && PYTHONPATH=/root/repo/baseline/_ref:/root/repo:/root/repo/tests CGB_KEY_SEED=0 timeout 1800 python -m pytest -q -p ref_dropin_plugin -p no:cacheprovider --rootdir . -o addopts= . --durations=12 > /root/repo/gpurun_out/ref_suite_all.log 2>&1; echo "all rc=$?"; tail -25 /root/repo/gpurun_out/ref_suite_all.log; cd /root/repo
for e in "CGB_KSROW8=1" ; do
env $e timeout 1200 python -m pytest tests/test_gpu_ring_parity.py tests/test_gpu_hotpath.py -q -x 2>&1 | tail -1
done
for e in "CGB_KSROW8=0" "CGB_KSROW8=1"; do for rep in 1 2; do
env $e timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$e', round(d['value'],2), round(d['e2e']['value'],2), {k:v['ms'] for k,v in list(d['units'].items())[:2]}, {k:d['kernels'][k]['ms'] for k in ('ks_row_md','ks_modup_cols','ks_row_P') if k in d['kernels']})"
done; done
