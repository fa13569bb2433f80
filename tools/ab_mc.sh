# A/B of the multi-crop launches: in-tree build vs ab/*.so on the same box
echo "tree"; python tools/time_mc.py 2>/dev/null | tail -4
for f in ab/*.so; do echo "$(basename $f)"; PF_B200_LIB=$PWD/$f python tools/time_mc.py 2>/dev/null | tail -4; done
