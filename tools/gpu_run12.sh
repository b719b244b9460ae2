timeout 300 python tools/cfg_lat.py
RNSW_K4_TWO_PASS=1 timeout 300 python tools/cfg_lat.py
