# Ozaki-product profiles at the current code: launch list of one map sequence at N=32768
# and full captures of the INT8 GEMM and the reconstruction at N=16384.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out
python tools/probes/ozaki_only.py 32768 3 > $O/oz_only.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/oz_launches.csv python tools/probes/ozaki_only.py 32768 1 > $O/oz_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:i8gemm -s 20 -c 1 -o $O/oz_i8gemm python tools/probes/ozaki_only.py 16384 2 > $O/oz_i8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:reconstruct -c 1 -o $O/oz_reconstruct python tools/probes/ozaki_only.py 16384 1 > $O/oz_rec.log 2>&1
cat $O/oz_only.txt
