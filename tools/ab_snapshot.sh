# Snapshot the currently built package (Python files + .so) under ab/<name>/ for A/B timing
# of engine variants in one GPU call: python tools/ab_time.py --pkg ab/<name> ...
set -e
name="$1"
root="$(cd "$(dirname "$0")/.." && pwd)"
rm -rf "$root/ab/$name"
mkdir -p "$root/ab/$name/paper_2403_03772_b200"
cp "$root"/paper_2403_03772_b200/*.py "$root"/paper_2403_03772_b200/*.so "$root/ab/$name/paper_2403_03772_b200/"
echo "snapshot ab/$name"
