cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for g in 4 6 8 10 12; do IPT_I8_GROUP=$g python tools/probes/ozaki_only.py 32768 3; done > $O/oz_group.txt 2>&1
cat $O/oz_group.txt
