# A/B: ReLU folded into the bf16 conversion (cvt.rn.relu.bf16x2.f32) vs fp32 max before converting
B='from paper_2506_22175_b200 import build; build.build(force=True)'
MPM_NVCC_FLAGS=-DMPM_RELU_CVT=0 python -c "$B" > gpurun_out/r2relu_build0.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_old.so
MPM_NVCC_FLAGS= python -c "$B" > gpurun_out/r2relu_build1.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_new.so
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -x > gpurun_out/r2relu_tests.log 2>&1; tail -2 gpurun_out/r2relu_tests.log
for r in 1 2 3; do for v in old new; do
  echo "== $v round$r" >> gpurun_out/r2relu.txt
  MPM_LIB=/tmp/libmpm_$v.so python tools/gemm_table.py --sustained --only cfg2_N1 --gemm fc1_fwd,fc2_dgrad >> gpurun_out/r2relu.txt 2>&1
  MPM_LIB=/tmp/libmpm_$v.so python bench.py --no-memory-sweep --no-cpu-baseline --pipeline-n 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['gemm_ms_per_step'])" >> gpurun_out/r2relu.txt 2>&1
done; done
python - <<'P'
import json
for l in open('gpurun_out/r2relu.txt'):
    if l.startswith('{'):
        d=json.loads(l); print(d['gemm'], round(d['ours_us'],1), round(d['ours_sustained_us'],1))
    else: print(l.strip())
P
