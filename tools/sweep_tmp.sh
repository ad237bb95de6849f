LGP_CG_VEC_TRACE=1 timeout 300 python tools/cg_periter.py cfg4 2>&1 | tail -9
timeout 300 python tools/cg_periter.py cfg3 cfg2 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_fullsize.py tests/test_gpu_loopback.py tests/test_gpu_errors.py tests/test_gpu_models.py -x -q 2>&1 | tail -3
bash tools/ncu_cg_launches_warm.sh cfg4 > gpurun_out/cgw.txt 2>&1; head -4 gpurun_out/cgw.txt
bash tools/ncu_cg_launches.sh cfg4 > gpurun_out/cgc.txt 2>&1; head -4 gpurun_out/cgc.txt
