python tools/sweep.py c1 '' 'EMPC_SMALL_THREADS=128' 'EMPC_SMALL_THREADS=256'
timeout 900 python -m pytest tests -q -m gpu --timeout 400 2>&1 | tail -2
