# compute-sanitizer memcheck on each rank of a 2-process peer-memory step (compacted dispatch / combine
# push for no reuse; ring pulls for S4): every worker process wrapped by its own sanitizer
mkdir -p gpurun_out/san
export MASTER_ADDR=127.0.0.1 WORLD_SIZE=2
port=29801
for strat in none s4; do
  export MASTER_PORT=$port
  for r in 0 1; do
    RANK=$r LOCAL_RANK=$r timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tests/p2p_worker.py \
      --out /tmp/san_$strat.npz --chunks 2 --strategy $strat --steps 1 > gpurun_out/san/r2_memcheck_p2p_${strat}_rank$r.log 2>&1 &
  done
  wait
  port=$((port + 1))
done
grep -H "ERROR SUMMARY" gpurun_out/san/r2_memcheck_p2p_*_rank*.log
