# A/B: epilogue warps issuing their TMEM loads together (named barrier) vs independently
B='from paper_2506_22175_b200 import build; build.build(force=True)'
MPM_NVCC_FLAGS= python -c "$B" > gpurun_out/r2sync_build0.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_a.so
MPM_NVCC_FLAGS=-DMPM_EPI_SYNC python -c "$B" > gpurun_out/r2sync_build1.log 2>&1; cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_b.so
for r in 1 2; do for v in a b; do
  echo "== $v round$r" >> gpurun_out/r2sync.txt
  MPM_LIB=/tmp/libmpm_$v.so python tools/gemm_table.py --sustained --only cfg2_N1 --gemm fc1_fwd,fc2_dgrad,fc2_wgrad >> gpurun_out/r2sync.txt 2>&1
done; done
python - <<'P'
import json
for l in open('gpurun_out/r2sync.txt'):
    if l.startswith('=='): print(l.strip()); continue
    if l.startswith('{'):
        d=json.loads(l); print(d['gemm'], round(d['ours_us'],1), round(d['ours_sustained_us'],1), d['ours_sustained_mhz'])
P
