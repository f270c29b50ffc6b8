# ncu full capture (source-level) of the default float matchers, after plain runs exit 0; exports
# the raw metrics and the source page as CSV on the box (reports removed: gpurun_out <= 64 MiB)
mkdir -p gpurun_out
rm -f gpurun_out/prof_f_status.txt
for c in ${CONFIGS:-c2 c3 c4}; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu ${EXTRA}"
  timeout 300 $B > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-bm_boxf}" -s 1 -c 1 -o /tmp/prof_f_$c $B > gpurun_out/ncu_f_$c.log 2>&1
  echo "$c=$?" >> gpurun_out/prof_f_status.txt
  ncu -i /tmp/prof_f_$c.ncu-rep --page raw --csv > gpurun_out/prof_f_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_f_$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_f_${c}_src.csv 2>/dev/null
  ncu -i /tmp/prof_f_$c.ncu-rep --page details --csv > gpurun_out/prof_f_${c}_details.csv 2>/dev/null
  gzip -f gpurun_out/prof_f_${c}_src.csv
done
