python tools/gpu/capability_runs.py > gpurun_out/capability_plain.json 2> gpurun_out/capability_plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/capability_ncu.csv python tools/gpu/capability_runs.py > gpurun_out/capability_ncu.log 2>&1
echo rc=$?
