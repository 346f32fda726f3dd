# register / occupancy variants of the K1 walk (config 5, 2,048 scenarios per call)
for v in default m6 m7 nb0 nb8; do
  if [ $v = default ]; then unset LUMOS_B200_LIB; else export LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_$v.so; fi
  python tools/walk_probe.py config5 2048 4 $v
done
