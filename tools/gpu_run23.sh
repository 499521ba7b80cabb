timeout 300 python tools/coldseq.py
