# compute-sanitizer on the round-2 kernels: the layer step (routing epilogue GEMM, zero-row groups) and a
# 2-process peer-memory step (compacted dispatch / combine push / ring pull)
mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_step.py > gpurun_out/san/r2_memcheck.log 2>&1; echo rc=$? >> gpurun_out/san/r2_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_step.py > gpurun_out/san/r2_synccheck.log 2>&1; echo rc=$? >> gpurun_out/san/r2_synccheck.log
for strat in none s4; do
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29791 tests/p2p_worker.py --out /tmp/san_$strat.npz --chunks 2 --strategy $strat --steps 1 > gpurun_out/san/r2_memcheck_p2p_$strat.log 2>&1; echo rc=$? >> gpurun_out/san/r2_memcheck_p2p_$strat.log
done
tail -3 gpurun_out/san/*.log
