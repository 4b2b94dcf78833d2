# GEMM evidence vs cuBLAS (energy, steady state, ncu counters) and the step's kernel timeline
python tools/kernel_timeline.py --n 2 --json gpurun_out/r2o_timeline_n2.json > gpurun_out/r2o_timeline_n2.txt 2>&1
python tools/kernel_timeline.py --n 1 --json gpurun_out/r2o_timeline_n1.json > gpurun_out/r2o_timeline_n1.txt 2>&1
python tools/gemm_table.py --sustained --out gpurun_out/r2o_gemm_vs_cublas_energy.json > gpurun_out/r2o_gemm_table.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"nvjet|gemm|umma" -o gpurun_out/r2o_cublas_vs_ours python tools/cublas_ncu_probe.py > gpurun_out/r2o_ncu.log 2>&1
