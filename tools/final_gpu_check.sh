cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r02}_final_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG:-r02}_final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG:-r02}_final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG:-r02}_final_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG:-r02}_final_bench_ref.log 2>&1
tail -3 gpurun_out/${TAG:-r02}_final_gpu_tests.log; cat gpurun_out/${TAG:-r02}_final_smoke.log | tail -2; tail -1 gpurun_out/${TAG:-r02}_final_bench.log | cut -c1-600
