timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "resnet or config5" 2>&1 | tail -15
timeout 300 python tools/resnet_probe.py
