timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gputest_r02.log
cat gpurun_out/gputest_r02.log
