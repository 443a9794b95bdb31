cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== pdl"; timeout 300 python scripts/gap_probe.py 89,148
echo "== nopdl"; SEMIPD_NO_PDL=1 timeout 300 python scripts/gap_probe.py 89,148
