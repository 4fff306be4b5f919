#!/bin/bash
# dump one kernel's SASS: tools/kernel_sass.sh <so> <mangled-name substring> > out.sass
d=$(mktemp -d)
so=$(realpath "$1")
(cd "$d" && cuobjdump -xelf all "$so" >/dev/null)
for c in "$d"/*.cubin; do
  cuobjdump -sass "$c" | awk -v k="$2" '/Function : /{f=index($0,k)>0} f'
done
rm -rf "$d"
