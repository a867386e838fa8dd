./tools/micro/zwide
python -m pytest tests/test_gpu_zfullsize.py "tests/test_gpu_parity.py::test_closed_form_constant_V" -x -q --durations=10 2>&1 | tail -25
