# codec 3 vs codec 4 (and any tools/diag_build.sh variants named in VARS) on
# the mu = 64 expert FFN microbenchmark
python tools/profile_kernels.py --mu 64 --only expert --codec3 2>&1 | grep -v "^{" | sed 's/^/codec3   /'
for v in base $VARS; do
  [ "$v" = "base" ] && v=""
  L=$PWD/paper_2411_11217_b200/libmlt${v:+_$v}.so
  MLT_LIB=$L python tools/profile_kernels.py --mu 64 --only expert --codec4 2>&1 | grep -v "^{" | sed "s/^/codec4${v:+_$v}   /"
done
