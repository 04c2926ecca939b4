#!/bin/bash
# Regenerates the io.hpp goldens with the unmodified reference headers
# (needs /root/reference; run in the build container).
set -e
cd "$(dirname "$0")"
g++ -std=c++20 -O1 -I /root/reference/proj/include gen_io.cpp -o /tmp/gen_io
/tmp/gen_io .
