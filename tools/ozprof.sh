cd "$GRAFT_REPO_ROOT"; O=gpurun_out
python tools/i8_probe.py > $O/i8_probe.txt 2>&1
python tools/ozaki_probe.py 8192 32768 > $O/oz_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/oz_launches.csv python tools/ozaki_only.py 32768 > $O/oz_l.log 2>&1
for k in i8gemm reconstruct residues; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/oz_$k python tools/ozaki_only.py 16384 > $O/oz_$k.log 2>&1
done
ls -la $O
