# sweep the fused x-plane kernel chunking on cfg2 / cfg5 / cfg3
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "fused or steps_match or config1 or flags" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -1 gpurun_out/pytest_gpu.log
for cfg in cfg2 cfg5 cfg3; do
for ch in 2048 4608 9216 18432; do for sm in 40960 57344 114688; do
  r=$(VPB_XPLANE_CHUNK=$ch VPB_XPLANE_SMEM=$sm timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['kernels']['sweep_x12']['avg_ms'],3), round(d['ms_per_step'],3))")
  echo "$cfg chunk=$ch smem=$sm -> x12_ms step_ms: $r"
done; done; done
