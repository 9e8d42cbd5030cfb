# large-sample index parity vs the oracle (CPU oracle runs in 16 processes? no: single process; bounded)
python tools/index_parity.py 2048 32 random smooth
python tools/index_parity.py 2048 32 trained smooth
python tools/index_parity.py 1024 32 random noise
python tools/index_parity.py 256 64 random smooth
python tools/index_parity.py 256 64 trained smooth
