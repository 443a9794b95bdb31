cd /root/repo
TL_B=256 TL_CTX=350 TL_OUT=tl_mla_350_104.json timeout 600 python scripts/timeline_mla.py 104 > gpurun_out/tl_mla_350.log 2>&1
TL_B=256 TL_CTX=350 TL_CTA=5 TL_OUT=tl_mla_350_104_c5.json timeout 600 python scripts/timeline_mla.py 104 >> gpurun_out/tl_mla_350.log 2>&1
tail -5 gpurun_out/tl_mla_350.log
