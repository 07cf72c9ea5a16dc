# usage: bisect_small.sh "<N B M [prec]>" name...  (name "cur" = the current build)
G=$1; shift
for N in "$@"; do
  if [ $N = cur ]; then E=""; else E="XKNN_PKG_DIR=ab/$N"; fi
  env $E timeout 120 python tools/step_small.py $G > /tmp/o_$N.txt 2>&1; echo "$N [$G] rc=$? $(tail -1 /tmp/o_$N.txt)"
done
