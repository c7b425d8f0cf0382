python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for c in 3 4 5 2; do timeout 200 python tools/quick_time.py $c 2>&1 | grep -E "^iter 3|^sha"; done
