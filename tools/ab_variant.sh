# A/B variants that differ in a few TUs only: ab_variant.sh "tu1.cu tu2.cu" name "flags" [name "flags" ...]
set -e
mkdir -p ab
TUS="$1"; shift
while [ $# -ge 2 ]; do
  python -c "from paper_2509_19821_b200.build import build_variant; build_variant('ab/$1.so', '''$2''', '''$TUS'''.split())"
  shift 2
done
