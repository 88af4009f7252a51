# A/B: time kinds with the base build and the current build (env CUR_ENV applied), interleaved, same box
for rep in 1 2; do
  for lib in base cur; do
    if [ $lib = base ]; then
      TPO_LIB_PATH=paper_2506_13523_b200/libtpo_b200_base.so timeout 300 python tools/kind_timing.py 2>&1 | grep -E "${KINDS:-grid|fourier}" | grep -v '"L": 16' | sed "s/^/$lib /"
    else
      env $CUR_ENV timeout 300 python tools/kind_timing.py 2>&1 | grep -E "${KINDS:-grid|fourier}" | grep -v '"L": 16' | sed "s/^/$lib /"
    fi
  done
done
