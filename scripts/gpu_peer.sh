set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -k "peer" -x -q -p no:cacheprovider > gpurun_out/tests_peer.txt 2>&1; tail -30 gpurun_out/tests_peer.txt
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/tests_fast.txt 2>&1; tail -3 gpurun_out/tests_fast.txt
