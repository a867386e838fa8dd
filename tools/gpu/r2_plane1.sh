timeout 900 python -m pytest tests/test_gpu_plane.py -x -q 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_zfullsize.py 2>&1 | tail -15
