# A/B: L2 eviction priority on the GEMM output stores (evict_first / evict_last / none)
B='from paper_2506_22175_b200 import build; build.build(force=True)'
MPM_NVCC_FLAGS= python -c "$B" > gpurun_out/r2hint_build0.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_0.so
MPM_NVCC_FLAGS=-DMPM_STORE_HINT=1 python -c "$B" > gpurun_out/r2hint_build1.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_1.so
MPM_NVCC_FLAGS=-DMPM_STORE_HINT=2 python -c "$B" > gpurun_out/r2hint_build2.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_2.so
for r in 1 2; do for v in 0 1 2; do
  echo "== hint$v round$r" >> gpurun_out/r2hint.txt
  MPM_LIB=/tmp/libmpm_$v.so python tools/gemm_table.py --sustained --only cfg2_N1 >> gpurun_out/r2hint.txt 2>&1
done; done
for r in 1 2; do for v in 0 1 2; do
  echo "== hint$v bench round$r" >> gpurun_out/r2hint.txt
  MPM_LIB=/tmp/libmpm_$v.so python bench.py --no-memory-sweep --no-cpu-baseline --pipeline-n 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['gemm_ms_per_step'])" >> gpurun_out/r2hint.txt 2>&1
done; done
python - <<'P'
import json
for l in open('gpurun_out/r2hint.txt'):
    if l.startswith('{'):
        d=json.loads(l); print(d['gemm'], round(d['ours_us'],1), round(d['ours_sustained_us'],1))
    else: print(l.strip())
P
