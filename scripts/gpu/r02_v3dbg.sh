export CASCADE_LIB=build/var_V3/libcascade.so
python scripts/dbench.py 64 8 2>&1 | tail -5
python -m pytest tests -m gpu -q -x -k "test_decode_matches_oracle" 2>&1 | tail -15
