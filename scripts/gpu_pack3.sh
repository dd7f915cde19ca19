python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "packed or shard or peer" 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
