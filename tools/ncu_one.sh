# usage: bash tools/ncu_one.sh <tag> <command...>
# Plain run first (must exit 0), then one ncu --set full capture of the first
# band kernel launch after 3 warm-up launches; exports raw + source pages as
# CSV and drops the (large) .ncu-rep so gpurun_out stays small.
tag=$1; shift
"$@" > gpurun_out/plain_$tag.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-band_iter} -s ${NCU_SKIP:-3} -c 1 \
    -o /tmp/prof_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1 || exit 2
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv > gpurun_out/src_$tag.csv 2>/dev/null
ncu -i /tmp/prof_$tag.ncu-rep --page details > gpurun_out/details_$tag.txt 2>/dev/null
