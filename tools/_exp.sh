O=gpurun_out
rm -f $O/exp.log
ncu --set full --clock-control none --import-source on -k regex:"k_est_t|k_place_t" -s 4 -c 4 -o $O/pe_full -f \
    python tools/prof_eval.py 100000000 > $O/ncu_pe.log 2>&1; echo pe=$? >> $O/exp.log
ncu -i $O/pe_full.ncu-rep --page raw --csv > $O/pe_full_raw.csv 2>/dev/null
ncu -i $O/pe_full.ncu-rep --page details --csv > $O/pe_full_details.csv 2>/dev/null
