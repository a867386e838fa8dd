python tools/gpu/c2_prof.py > gpurun_out/c2plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -s 40 -c 6 --csv --log-file gpurun_out/c2_launches.csv python tools/gpu/c2_prof.py > gpurun_out/c2ncu.log 2>&1
echo rc=$?; grep -v "==PROF==" gpurun_out/c2_launches.csv | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>10 and r[0]!='ID': print(r[4][:40], r[-3], r[-1])"
