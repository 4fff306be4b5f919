#!/bin/bash
# count local-memory (spill) instructions in one kernel's SASS: tools/spills.sh <so> <mangled-name substring>
set -e
d=$(mktemp -d)
cd "$d" && cuobjdump -xelf all "$(realpath -m "$OLDPWD/$1")" >/dev/null
for c in *.cubin; do
  cuobjdump -sass "$c" | awk -v k="$2" '/Function : /{f=index($0,k)>0} f' | grep -cE "STL|LDL" || true
done | sort -n | tail -1
rm -rf "$d"
