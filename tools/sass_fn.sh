#!/bin/bash
# Print the SASS of one kernel instantiation from an object file:
#   bash tools/sass_fn.sh <file.o> <mangled-name-substring>
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/ {on = index($0, pat) > 0} on'
