#!/bin/bash
# Build libqtm_<tag>.so from the committed HEAD sources (tag "base") for A/B runs
set -e
cd $(dirname $0)/..
TMP=$(mktemp -d)
git show HEAD:paper_1810_03047_b200/csrc/qtm_traj.cuh > $TMP/qtm_traj.cuh
git show HEAD:paper_1810_03047_b200/csrc/qtm_capi.cu > $TMP/qtm_capi.cu
cp paper_1810_03047_b200/csrc/qtm_traj.cuh $TMP/cur_traj.cuh; cp paper_1810_03047_b200/csrc/qtm_capi.cu $TMP/cur_capi.cu
cp $TMP/qtm_traj.cuh paper_1810_03047_b200/csrc/qtm_traj.cuh; cp $TMP/qtm_capi.cu paper_1810_03047_b200/csrc/qtm_capi.cu
QTM_BUILD_TAG=base python -m paper_1810_03047_b200.build > /dev/null || true
cp $TMP/cur_traj.cuh paper_1810_03047_b200/csrc/qtm_traj.cuh; cp $TMP/cur_capi.cu paper_1810_03047_b200/csrc/qtm_capi.cu
python -m paper_1810_03047_b200.build > /dev/null
rm -rf $TMP
ls -la paper_1810_03047_b200/libqtm*.so
