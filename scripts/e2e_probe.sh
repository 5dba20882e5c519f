O=gpurun_out/e2e; mkdir -p $O
nproc > $O/nproc.txt; lscpu | head -20 >> $O/nproc.txt
timeout 300 python scripts/h2d_probe.py > $O/h2d.txt 2>&1
timeout 600 python scripts/prof_hist_e2e.py > $O/hist_e2e.txt 2>&1
cat $O/nproc.txt $O/h2d.txt $O/hist_e2e.txt
