for w in 16 24 32; do
  echo "=== EBC_WARPS_PER_SM=$w"
  EBC_NVCC_FLAGS="-DEBC_FEW_SHAPES -DEBC_WARPS_PER_SM=$w" python paper_1910_11039_b200/build.py --force > /dev/null 2>&1
  python tools/sweep_c2.py "128,4,0;128,2,0;64,4,0;256,4,0;256,2,0" 400000
done
