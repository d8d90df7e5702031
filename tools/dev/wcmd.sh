timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for i in 1 2; do python tools/time_config.py --config c3 --reps 20; python tools/time_config.py --config c4 --reps 10; done
