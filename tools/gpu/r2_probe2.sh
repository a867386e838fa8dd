./tools/micro/zblock
python tools/gpu/oracle_speed.py
