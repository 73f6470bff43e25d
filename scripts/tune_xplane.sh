# sweep the fused x-plane kernel launch parameters on cfg2 / cfg5
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "fused or steps_match or config1" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
for cfg in cfg2 cfg5; do
for th in 192 384 576; do for ch in 16384 32768; do for sm in 112640 225280; do
  r=$(VPB_XPLANE_THREADS=$th VPB_XPLANE_CHUNK=$ch VPB_XPLANE_SMEM=$sm timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['kernels']['sweep_x12']['avg_ms'],3), round(d['ms_per_step'],3))")
  echo "$cfg threads=$th chunk=$ch smem=$sm -> x12_ms step_ms: $r"
done; done; done; done
