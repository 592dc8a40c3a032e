OUT=gpurun_out/rbncu; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_csr_group<.*EpiRestrictBegin" -c 1 -o $OUT/prof_rb python tools/one_solve.py > $OUT/log 2>&1
echo done >> $OUT/status.txt
