#!/bin/bash
# build the library with extra compile flags into probes/lib_$1.so (A/B experiments:
# probes/ab.sh $1), then rebuild the default library
set -e
cd "$(dirname "$0")/.."
SMY_EXTRA_CFLAGS="$2" python -m paper_2503_10725_b200.build > /tmp/smy_build_$1.log 2>&1 || { grep -A6 error /tmp/smy_build_$1.log | head -20; exit 1; }
cp paper_2503_10725_b200/libsamoyeds.so probes/lib_$1.so
python -m paper_2503_10725_b200.build > /tmp/smy_build.log 2>&1
echo "built probes/lib_$1.so ($2)"
