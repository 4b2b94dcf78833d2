# epilogue cost A/B, part 3: TMEM loads only (skip4) against loads + math (skip2), nothing (skip3), full (skip0)
B='from paper_2506_22175_b200 import build; build.build(force=True)'
for v in 0 2 3 4; do
  if [ $v = 0 ]; then MPM_NVCC_FLAGS= python -c "$B"; else MPM_NVCC_FLAGS=-DMPM_EPI_SKIP=$v python -c "$B"; fi > gpurun_out/r2skip3_build$v.log 2>&1
  cp paper_2506_22175_b200/libmpm.so /tmp/libmpm_skip$v.so
done
for r in 1 2; do for v in 0 2 3 4; do
  echo "== skip$v round$r" >> gpurun_out/r2skip3.txt
  MPM_LIB=/tmp/libmpm_skip$v.so python tools/gemm_table.py --sustained --only cfg2_N1 --gemm fc1_fwd,fc2_dgrad,fc2_wgrad >> gpurun_out/r2skip3.txt 2>&1
done; done
python - <<'P'
import json
for l in open('gpurun_out/r2skip3.txt'):
    if l.startswith('=='): print(l.strip()); continue
    if l.startswith('{'):
        d=json.loads(l); print(d['gemm'], round(d['ours_us'],1), round(d['ours_sustained_us'],1), d['ours_sustained_mhz'])
P
