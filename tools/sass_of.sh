#!/bin/sh
# sass_of.sh LIB PATTERN — SASS of the first kernel whose mangled name matches PATTERN
cuobjdump -sass "$1" 2>/dev/null | awk -v pat="$2" '
  /Function :/ { on = ($0 ~ pat) ? 1 : 0; if (on) found++; if (found > 1) on = 0; next }
  on && /^[ \t]+\/\*[0-9a-f]{4}\*\// { sub(/\/\* 0x[0-9a-f]* \*\//, ""); print }'
