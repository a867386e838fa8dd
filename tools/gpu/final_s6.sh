# final check of the session: GPU suite, default bench, C4 bench, smoke
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.err
timeout 600 python bench.py --config C4 --no-solvers --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench C4 rc=$?"; tail -1 gpurun_out/bench_c4.err
python -c "
import json
for f in ('gpurun_out/bench_full.json', 'gpurun_out/bench_c4.json'):
    d = json.load(open(f)); print(f, d['value'], d['config']['iteration_form'], d['iteration_roofline'], d['roofline']['frac'], d['kernel_ms_per_launch'], d['clocks'], d['e2e']['value'] if d.get('e2e') else None)
"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
