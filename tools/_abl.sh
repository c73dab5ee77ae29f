python tools/build_rate.py
BATCH=262144 python tools/build_rate.py
