#!/bin/bash
# Build a variant of the library in a scratch copy (sed expression applied to
# one csrc file) and run a command from that copy: A/B of compile-time knobs.
#   tools/variant.sh <file> '<sed expr>' <command...>
set -e
f=$1; expr=$2; shift 2
V=/tmp/pk_variant; rm -rf $V; mkdir -p $V
cp -r paper_2312_03940_b200 include oracle tools $V/
sed -i "$expr" $V/paper_2312_03940_b200/csrc/$f
rm -f $V/paper_2312_03940_b200/libpeakann_b200.so; rm -rf $V/paper_2312_03940_b200/csrc/build
make -s -C $V/paper_2312_03940_b200/csrc > /dev/null 2>&1
cd $V && "$@"
