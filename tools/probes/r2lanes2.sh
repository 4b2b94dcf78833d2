# two compute lanes vs one at BASELINE configs[2] (M=2048, H=8192, E=32, top-1) near the lane gate
P="timeout 300 python tools/cfg4_probe.py --M 2048 --H 8192 --E 32 --k 1 --steps 10"
for r in 1 2; do for T in 32768 65536; do for n in 2 4; do
  $P --tokens $T --n $n >> gpurun_out/r2lanes2.jsonl 2>> gpurun_out/r2lanes2.err
  MPM_COMPUTE_LANES=1 $P --tokens $T --n $n >> gpurun_out/r2lanes2.jsonl 2>> gpurun_out/r2lanes2.err
done; done; done
python - <<'P'
import json
for l in open('gpurun_out/r2lanes2.jsonl'):
    d=json.loads(l); print(d['tokens'], d['n'], d['lanes'], d['ms_per_step'], d['clocks']['sm_mhz'])
P
tail -2 gpurun_out/r2lanes2.err
