# compute-sanitizer memcheck (one tool per call) on the small-grid kernel families
set -x
o=gpurun_out/r02b_san; mkdir -p $o
timeout 600 python scripts/sanitize.py dg advance spline plugin > $o/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python scripts/sanitize.py dg advance spline plugin > $o/memcheck.log 2>&1; echo rc=$? >> $o/memcheck.log
tail -5 $o/memcheck.log
