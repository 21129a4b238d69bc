#!/bin/sh
# Build the C oracle (test infrastructure; never linked by the product).
set -e
here=$(cd "$(dirname "$0")" && pwd)
mkdir -p "$here/build"
gcc -O2 -fopenmp -fPIC -shared -std=c11 -o "$here/build/libgconn_oracle.so" "$here/gconn_oracle.c" -lm
echo "$here/build/libgconn_oracle.so"
