for M in 103307 20663; do for v in 0 1 2; do echo "M=$M v=$v"; SFFTB_HASH_VARIANT=$v python tools/prof_hash.py 26 4 $M 2>&1 | tail -2; done; done
