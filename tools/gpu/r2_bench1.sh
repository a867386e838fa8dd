python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?
tail -c 3000 gpurun_out/bench1.err
