# configs[3] step time under A/B switches (round-2 memory sweep check)
P="timeout 300 python tools/cfg4_probe.py"
for r in 1 2; do
  $P --n 8 >> gpurun_out/r2cfg4.jsonl 2>> gpurun_out/r2cfg4.err
  MPM_COMPUTE_LANES=1 $P --n 8 >> gpurun_out/r2cfg4.jsonl 2>> gpurun_out/r2cfg4.err
  MPM_COMPACT=0 $P --n 8 >> gpurun_out/r2cfg4.jsonl 2>> gpurun_out/r2cfg4.err
  $P --n 1 >> gpurun_out/r2cfg4.jsonl 2>> gpurun_out/r2cfg4.err
done
cut -c1-400 gpurun_out/r2cfg4.jsonl; tail -3 gpurun_out/r2cfg4.err
