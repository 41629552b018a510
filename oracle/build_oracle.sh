#!/usr/bin/env bash
# Build the CPU oracle (test infrastructure only): oracle/_build/librsh_oracle.so
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
mkdir -p "$here/_build"
gcc -O2 -fPIC -fopenmp -shared -o "$here/_build/librsh_oracle.so" "$here/rsh_oracle.c"
