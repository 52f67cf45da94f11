# Fresh-box re-check of the multi-GPU paths at N = 4 (run with gpurun --gpus 4).
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -rs > gpurun_out/${TAG:-r02}_n4_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG:-r02}_n4_gpu_tests.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/${TAG:-r02}_n${n}_bench.log 2>&1
done
tail -3 gpurun_out/${TAG:-r02}_n4_gpu_tests.log; for n in 2 4; do tail -1 gpurun_out/${TAG:-r02}_n${n}_bench.log | cut -c1-300; done
