# full-length parity runs (tests/parity_fullsize.py), results in profiles/
nproc; free -g | head -2
python tests/parity_fullsize.py --configs C1,C2,C3,C4,C5 --out gpurun_out/parity_fullsize_r02.json
