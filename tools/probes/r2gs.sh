# sparse gate weight gradient from the routed assignments: parity tests, then bench A/B (MPM_GATE_SPARSE)
python -m pytest tests/test_gpu_kernels.py -x -q -k "gate" > gpurun_out/r2gs_tests.log 2>&1; echo rc=$? >> gpurun_out/r2gs_tests.log
for rep in 1 2; do
for v in "MPM_GATE_SPARSE=0" "X=0"; do
  env $v python bench.py --no-memory-sweep --no-cpu-baseline 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6, 3), round(d['ms_per_step'], 4), d['step_breakdown']['phases_ms']['bwd_combine_bwd'])"
done; done > gpurun_out/r2gs_bench.txt
python tools/hbm_probe.py 30 2>&1 | grep -E "gate_bwd_gemms|gate_wgrad_routed" > gpurun_out/r2gs_hbm.txt; python tools/kernel_timeline.py --n 1 > gpurun_out/r2gs_timeline_n1.txt 2>&1; cat gpurun_out/r2gs_hbm.txt
tail -2 gpurun_out/r2gs_tests.log; cat gpurun_out/r2gs_bench.txt
