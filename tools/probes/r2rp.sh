# gate GEMM + routing epilogue: single-CTA 128-row tiles vs 2-CTA pairs (MPM_ROUTE_PAIR), kernel and step
for rep in 1 2; do
for v in "MPM_ROUTE_PAIR=0" "X=0"; do
  env $v python tools/hbm_probe.py 30 2>&1 | grep gate_route | sed "s/^/$v /"
done; done > gpurun_out/r2rp.txt
python -m pytest tests/test_gpu_kernels.py -q -x -k "gate" > gpurun_out/r2rp_tests.log 2>&1; echo rc=$? >> gpurun_out/r2rp_tests.log
for rep in 1 2; do
for v in "MPM_ROUTE_PAIR=0" "X=0"; do
  env $v python bench.py --no-memory-sweep --no-cpu-baseline 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6, 3), round(d['ms_per_step'], 4), d['step_breakdown']['phases_ms']['fwd_routing_permute'])"
done; done > gpurun_out/r2rp_bench.txt
cat gpurun_out/r2rp.txt gpurun_out/r2rp_bench.txt; tail -2 gpurun_out/r2rp_tests.log
