#!/bin/bash
# Export the pages of an ncu report we read here (raw metrics + per-line source counters
# of each captured kernel) as CSV, then drop the (large) report.  Usage: ncu_export.sh rep.ncu-rep out_prefix
rep=$1; out=$2
ncu -i "$rep" --page raw --csv > "${out}_raw.csv" 2>/dev/null
ncu -i "$rep" --page details --csv > "${out}_details.csv" 2>/dev/null
n=$(ncu -i "$rep" --page raw --csv 2>/dev/null | tail -n +3 | wc -l)
for ((i=0; i<n; i++)); do
  ncu -i "$rep" --page source --csv --print-source cuda -s $i -c 1 > "${out}_src${i}_cuda.csv" 2>/dev/null
  ncu -i "$rep" --page source --csv --print-source sass -s $i -c 1 > "${out}_src${i}_sass.csv" 2>/dev/null
done
gzip -f "${out}"_src*_sass.csv
rm -f "$rep"
