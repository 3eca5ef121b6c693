cd "$GRAFT_REPO_ROOT"; O=gpurun_out
for g in 1000000 4 8 16; do IPT_I8_GROUP=$g python tools/ozaki_only.py 32768 3; done > $O/oz_group.txt 2>&1
for g in 8 16; do IPT_I8_GROUP=$g IPT_I8_KERNEL=2sm python tools/ozaki_only.py 32768 3; done >> $O/oz_group.txt 2>&1
IPT_I8_GROUP=8 ncu --set full --clock-control none -k regex:i8gemm -s 20 -c 1 -o $O/oz_i8gemm_g8 python tools/ozaki_only.py 16384 2 > $O/oz_i8g.log 2>&1
cat $O/oz_group.txt
