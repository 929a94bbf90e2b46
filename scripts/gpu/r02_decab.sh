for v in base NOCHECK V3; do
  if [ $v = base ]; then unset CASCADE_LIB; else export CASCADE_LIB=build/var_$v/libcascade.so; fi
  echo "== $v"; python scripts/dbench.py 64 32 2>&1 | tail -1
done
