# where the expert GEMMs' warp roles wait: probe build of libmpm (clock64 sums per role)
MPM_NVCC_FLAGS=-DMPM_EPI_PROBE python -c "from paper_2506_22175_b200 import build; build.build(force=True)" > gpurun_out/r2epi_build.log 2>&1
python tools/epi_probe.py > gpurun_out/r2epi_probe.jsonl 2> gpurun_out/r2epi_probe.err
python tools/epi_probe.py fc1_fwd,fc2_fwd,fc1_dgrad >> gpurun_out/r2epi_probe.jsonl 2>> gpurun_out/r2epi_probe.err
cat gpurun_out/r2epi_probe.jsonl; tail -3 gpurun_out/r2epi_probe.err
