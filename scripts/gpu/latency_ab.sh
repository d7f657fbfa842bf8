#!/bin/bash
# config 1 latency from C (scripts/latency.cpp) for two builds of the library
# usage: latency_ab.sh <libA.so> <libB.so> [calls]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for L in "$1" "$2"; do
  d=$(mktemp -d); cp "$L" "$d/libdespot.so"
  g++ -O2 -std=c++17 scripts/latency.cpp -Iinclude -I/usr/local/cuda/include -L"$d" -ldespot \
    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,"$d" -o "$d/latency" && echo "$L" && "$d/latency" "${3:-3000}" | cut -c1-60
done
