#!/bin/bash
# build the library; print the error tail and fail if the build fails
cd "$(dirname "$0")/.." && python -m paper_2503_10725_b200.build > /tmp/smy_build.log 2>&1 && echo "build ok" || { grep -A6 "error" /tmp/smy_build.log | head -30; exit 1; }
