"""Host build of the kernel's pure helpers (csrc/bits.cuh): column compression
and the per-biclique hash, checked against plain definitions."""
import os
import subprocess

import pytest

from oracle import reference as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r"""
#include <cstdio>
#include <cstdint>
#include "bits.cuh"
static uint64_t s = 88172645463325252ull;
static uint64_t rnd() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main() {
  int bad = 0;
  // compress vs bit-by-bit definition, W = 1, 2, 4
  for (int it = 0; it < 200000; ++it) {
    uint32_t m[4], x[4], out[4], ref[4] = {0, 0, 0, 0};
    int W = it % 3 == 0 ? 1 : (it % 3 == 1 ? 2 : 4);
    for (int w = 0; w < 4; ++w) { m[w] = (uint32_t)rnd(); x[w] = (uint32_t)rnd();
      if (it % 7 == 0) m[w] = 0; if (it % 11 == 0) m[w] = 0xffffffffu; }
    int k = 0;
    for (int w = 0; w < W; ++w) for (int b = 0; b < 32; ++b) if (m[w] >> b & 1) {
      if (x[w] >> b & 1) ref[k >> 5] |= 1u << (k & 31);
      ++k;
    }
    if (W == 1) { auto c = mbe_compress_prep_w<1>(m); mbe_compress_apply_w<1>(c, x, out); }
    else if (W == 2) { auto c = mbe_compress_prep_w<2>(m); mbe_compress_apply_w<2>(c, x, out); }
    else { auto c = mbe_compress_prep_w<4>(m); mbe_compress_apply_w<4>(c, x, out); }
    for (int w = 0; w < 4; ++w) if (out[w] != ref[w]) { ++bad; break; }
  }
  printf("compress_bad %d\n", bad);
  // hash of a biclique given side sums
  printf("mix %llu %llu\n", (unsigned long long)mbe_mix64(0), (unsigned long long)mbe_mix64(12345));
  uint64_t sL = mbe_mix64(2 * 3 + 1) + mbe_mix64(2 * 5 + 1);           // L' = {3, 5} on side 2
  uint64_t sR = mbe_mix64(2 * 0) + mbe_mix64(2 * 7) + mbe_mix64(2 * 9);  // R' = {0, 7, 9} on side 1
  printf("h1 %llu\n", (unsigned long long)mbe_biclique_hash(1, sL, 2, sR, 3));
  uint64_t sL2 = mbe_mix64(2 * 0) + mbe_mix64(2 * 7) + mbe_mix64(2 * 9);  // cand side 2: L' on side 1
  uint64_t sR2 = mbe_mix64(2 * 3 + 1) + mbe_mix64(2 * 5 + 1);
  printf("h2 %llu\n", (unsigned long long)mbe_biclique_hash(2, sL2, 3, sR2, 2));
  printf("words %u %u %u %u %u\n", mbe_words_for(1), mbe_words_for(32), mbe_words_for(33), mbe_words_for(64),
         mbe_words_for(65));
  return 0;
}
"""


@pytest.fixture(scope="module")
def out(tmp_path_factory):
    d = tmp_path_factory.mktemp("bits")
    src = d / "t.cpp"
    src.write_text(PROG)
    exe = d / "t"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2401_05039_b200", "csrc"),
                           str(src), "-o", str(exe)])
    return dict((line.split()[0], line.split()[1:]) for line in subprocess.check_output([str(exe)]).decode().splitlines())


def test_compress_matches_definition(out):
    assert out["compress_bad"] == ["0"]


def test_library_hash_matches_definition(out):
    assert int(out["mix"][0]) == R.mix64(0)
    assert int(out["mix"][1]) == R.mix64(12345)
    assert int(out["h1"][0]) == R.biclique_hash((0, 7, 9), (3, 5))
    assert int(out["h2"][0]) == R.biclique_hash((0, 7, 9), (3, 5))


def test_words_for(out):
    assert out["words"] == ["1", "1", "2", "2", "4"]
