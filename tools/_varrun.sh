for v in base ne g74 g74ne g36ne; do
  if [ $v = base ]; then L=""; else L="ZT_LIB_PATH=build_var/$v/libzt.so"; fi
  echo "== $v"; env $L timeout 120 python tools/oz_modgemm_time.py 2048
done
