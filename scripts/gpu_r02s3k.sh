cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in base flip base flip; do
  PICO_LIB=build_variants/libpico_$v.so timeout 600 python scripts/po_profile.py T > gpurun_out/s3k_po_T_$v.txt 2>&1
  echo $v; sed -n 3,5p gpurun_out/s3k_po_T_$v.txt | cut -c1-400
done
