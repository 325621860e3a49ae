set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_2602_08798_b200._native as n; n.build(verbose=True)"
timeout 600 python -m pytest tests/test_gpu_primitives.py -x -q 2>&1 | tail -30
