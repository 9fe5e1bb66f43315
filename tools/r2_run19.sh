python -m pytest tests/test_gpu_symmetric.py -q -m gpu -x --durations=8 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'sym', d['symmetric_mode'], 'roof', d['roofline']['frac'], d['roofline']['kernel'][:60])"
