bash tools/build_probe.sh >/dev/null 2>&1 || echo build failed
ls tools/ablib/
for rep in 1 2; do
  for b in tools/ablib/sweep_probe_base tools/sweep_probe; do
    echo "== $b"
    $b 30 20 0 custom 3 12 0x7; $b 30 20 2 custom 3 12 0x7
    $b 30 100 0 9; $b 30 100 0 0
  done
done
tools/sweep_probe check 13 22 2 2>&1 | grep -E "FAIL|check" | tail -3
CFG=30:10 ITERS=10 bash tools/ab_r2.sh
python -m pytest tests/test_gpu_parity.py tests/test_gpu_symmetric.py tests/test_gpu_layout_swap.py -q -m gpu -x 2>&1 | tail -2
