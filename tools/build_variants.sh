# build libfrb200 variants with extra -D flags: build_variants.sh name "-DX=1" name2 "-DY=2" ...
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  python -c "import sys, __graft_entry__ as g; g.build(defines=tuple(sys.argv[2].split()), lib='paper_2305_07030_b200/lib/libfrb200_' + sys.argv[1] + '.so')" "$name" "$flags" &
done
wait
ls -la paper_2305_07030_b200/lib/
