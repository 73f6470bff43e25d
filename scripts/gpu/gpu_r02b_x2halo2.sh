# x1 x x2 stencil passes: the GPU dist tests after the parameter fix
set -x
o=gpurun_out/r02b_x2h2; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guards.py -m gpu -q -p no:cacheprovider > $o/pytest_dist.log 2>&1; echo rc=$? >> $o/pytest_dist.log
ls $o
