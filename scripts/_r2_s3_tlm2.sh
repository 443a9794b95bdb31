cd /root/repo
TL_B=64 TL_CTX=4000 TL_OUT=tl_mla_b64c4000.json timeout 600 python scripts/timeline_mla.py 104 2>&1 | tail -3
TL_B=256 TL_CTX=1000 TL_OUT=tl_mla_b256c1000.json timeout 600 python scripts/timeline_mla.py 104 2>&1 | tail -3
