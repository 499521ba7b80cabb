timeout 300 python tools/perblock.py
