# Build a library variant into paper_2509_13523_b200/_build_variants/NAME.so for A/B runs (SWF_LIB).
# usage: bash tools/build_variant.sh NAME [GIT_REV] [EXTRA nvcc flags]
#   GIT_REV: take csrc/ from that revision instead of the working tree (e.g. HEAD)
set -e
NAME=$1; REV=${2:-}; EXTRA=${3:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TOP=$(mktemp -d)
TMP=$TOP/pkg
mkdir -p $TMP
ln -s "$ROOT/include" "$TOP/include"
cp -r "$ROOT/paper_2509_13523_b200/csrc" "$ROOT/paper_2509_13523_b200/Makefile" "$TMP/"
if [ -n "$REV" ]; then
  (cd "$ROOT" && git archive "$REV" paper_2509_13523_b200/csrc) | tar -x -C "$TMP" --strip-components=1
fi
mkdir -p "$ROOT/paper_2509_13523_b200/_build_variants"
make -s -j8 -C "$TMP" NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include $EXTRA" >/dev/null
cp "$TMP/_build/libswinflow_b200.so" "$ROOT/paper_2509_13523_b200/_build_variants/$NAME.so"
rm -rf "$TOP"
echo "built _build_variants/$NAME.so"
