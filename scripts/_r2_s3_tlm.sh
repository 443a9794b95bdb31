cd /root/repo
for b in 104 148; do
TL_LOGN=1 TL_CTX=350 TL_OUT=tl_mla_logn_$b.json timeout 600 python scripts/timeline_mla.py $b 2>&1 | tail -4
done
TL_CTA=5 TL_LOGN=1 TL_CTX=350 TL_OUT=tl_mla_logn_148_c5.json timeout 600 python scripts/timeline_mla.py 148 2>&1 | tail -3
