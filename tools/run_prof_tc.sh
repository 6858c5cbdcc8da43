for dbg in 4 6; do echo "dbg$dbg"; SFFTB_HASH_TC_DBG=$dbg SFFTB_HASH_TC_SW=16 timeout 60 python tools/prof_hash.py 26 3 2>&1 | grep -v checks; done
echo "dbg4 nomc"; SFFTB_HASH_TC_NOMC=1 SFFTB_HASH_TC_DBG=4 SFFTB_HASH_TC_SW=16 timeout 60 python tools/prof_hash.py 26 3 2>&1 | grep -v checks
echo "dbg6 nomc"; SFFTB_HASH_TC_NOMC=1 SFFTB_HASH_TC_DBG=6 SFFTB_HASH_TC_SW=16 timeout 60 python tools/prof_hash.py 26 3 2>&1 | grep -v checks
echo "dbg6 nomc sw128"; SFFTB_HASH_TC_NOMC=1 SFFTB_HASH_TC_DBG=6 SFFTB_HASH_TC_SW=128 timeout 60 python tools/prof_hash.py 26 3 2>&1 | grep -v checks
echo "trace dbg6 nomc"; SFFTB_HASH_TC_NOMC=1 SFFTB_HASH_TC_DBG=6 SFFTB_HASH_TC_SW=16 SFFTB_HASH_TC_TRACE=1 timeout 60 python tools/prof_hash.py 24 1 2>&1 | head -24
