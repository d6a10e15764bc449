#!/bin/bash
# usage: tools/sass_of.sh '<demangled substring>' [lib]  -> SASS of the first matching kernel
lib=${2:-paper_2407_01943_b200/lib/libnus_b200.so}
sym=$(cuobjdump -res-usage "$lib" 2>/dev/null | grep -o "Function [^:]*" | awk '{print $2}' | while read m; do d=$(echo "$m" | c++filt); case "$d" in *"$1"*) echo "$m"; break;; esac; done)
[ -z "$sym" ] && { echo "no kernel matches $1" >&2; exit 1; }
cuobjdump -sass -fun "$sym" "$lib"
