for nq in 256 512 1024 4096; do
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:match_tc -s 2 -c 1 python scripts/die_probe.py $nq 2>/dev/null | grep -E "dram__bytes|gpu__time|plan|splits"
done
