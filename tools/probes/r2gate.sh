# gate GEMM + routing epilogue: where its warp roles wait (probe build)
MPM_NVCC_FLAGS=-DMPM_EPI_PROBE python -c "from paper_2506_22175_b200 import build; build.build(force=True)" > gpurun_out/r2gate_build.log 2>&1
python tools/epi_probe.py gate_route > gpurun_out/r2gate_probe.jsonl 2> gpurun_out/r2gate_probe.err
python tools/epi_probe.py gate_bwd >> gpurun_out/r2gate_probe.jsonl 2>> gpurun_out/r2gate_probe.err
cat gpurun_out/r2gate_probe.jsonl; tail -3 gpurun_out/r2gate_probe.err
