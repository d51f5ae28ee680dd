// qt_device.cuh -- small device helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qtb {

// XOR swizzle of 16-B smem slots: folds every higher 3-bit group of the
// index onto the low 3 bits so lanes that differ in (almost any) three tile
// bits land in distinct 16-B bank groups. Linear over GF(2):
// swz(a | b) == swz(a) ^ swz(b) for disjoint a, b.
__device__ __forceinline__ uint32_t swz(uint32_t j) {
  return j ^ ((j >> 3) & 7u) ^ ((j >> 6) & 7u) ^ ((j >> 9) & 7u) ^
         ((j >> 12) & 7u);
}

// software parallel-bit-deposit: bit i of x goes to the i-th set bit of mask
__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t b = 1; mask; b <<= 1) {
    const uint64_t low = mask & (~mask + 1);
    if (x & b) r |= low;
    mask ^= low;
  }
  return r;
}

__device__ __forceinline__ uint32_t insert_zero(uint32_t x, uint32_t p) {
  return ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u));
}

__device__ __forceinline__ bool finite2(double2 v) {
  // exponent all-ones <=> inf/nan; integer test keeps the FP64 pipe free
  const uint32_t hx = __double2hiint(v.x), hy = __double2hiint(v.y);
  return ((hx & 0x7ff00000u) != 0x7ff00000u) &&
         ((hy & 0x7ff00000u) != 0x7ff00000u);
}

__device__ __forceinline__ double2 neg2(double2 v) {
  // sign flip with integer ops (no FP64 instruction)
  return make_double2(
      __hiloint2double(__double2hiint(v.x) ^ 0x80000000, __double2loint(v.x)),
      __hiloint2double(__double2hiint(v.y) ^ 0x80000000, __double2loint(v.y)));
}

__device__ __forceinline__ double2 cmulz(double2 a, double br, double bi) {
  return make_double2(a.x * br - a.y * bi, a.x * bi + a.y * br);
}

}  // namespace qtb
