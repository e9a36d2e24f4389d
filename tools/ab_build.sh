# builds A/B variants of the engine library: ab_build.sh name "-DFLAG=1 ..." [name "flags" ...]
# (each a full rebuild into ab/<name>.so; the default build is restored last)
set -e
mkdir -p ab
while [ $# -ge 2 ]; do
  GMPEA_NVCC_EXTRA="$2" python -c "from paper_2509_19821_b200.build import build; build(force=True)"
  cp paper_2509_19821_b200/libgmpea_b200.so ab/$1.so
  shift 2
done
python -c "from paper_2509_19821_b200.build import build; build(force=True)"
