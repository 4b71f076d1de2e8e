set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_optimizer.py -q -x 2>&1 | tail -25
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -30
