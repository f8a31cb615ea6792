// mlp_common.cuh -- device helpers shared by the MLP kernels (mlp_l1/l2/sm100.cu):
// packed-bf16x2 GELU, fp32->bf16x2 packing, UMMA descriptors, TMA stores and
// the 128-byte-swizzled staging layout the TMA store/load maps use.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace rcm {

// GELU of the bf16 path, tanh form 0.5 x (1 + tanh(x (c0 + c1 x^2))), c0 = sqrt(2/pi),
// c1 = 0.044715 c0, evaluated in packed f16x2 arithmetic (one MUFU tanh per element) on the
// accumulator parked as f16 pairs, then rounded ONCE to bf16.  f16 carries 11 significant bits,
// so the pre-GELU parking and the GELU arithmetic add ~2^-11 relative error against the 2^-9 of
// the single bf16 output rounding: measured in emulation (tests/_emulate.py, R17) this
// sits within 3% of an exact-erf fp32 GELU with one rounding, where the round-1 bf16x2 arithmetic
// (accumulator rounded to bf16 before GELU, every op in bf16) was 1.3-1.6x the rounding floor.
// Range: inputs are parked with .satfinite (|x| <= 65504); x^2 or the tanh argument overflowing
// to +-inf gives tanh = +-1, i.e. GELU = x or 0, the correct limits.
__device__ __forceinline__ uint32_t cvt_f16x2(float lo, float hi) {  // .satfinite: range guard
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t f16x2_to_bf16x2(uint32_t v) {  // exact widen, one RNE rounding
  uint32_t r;
  asm("{\n\t.reg .f16 l, h;\n\t.reg .f32 fl, fh;\n\tmov.b32 {l, h}, %1;\n\tcvt.f32.f16 fl, l;\n\t"
      "cvt.f32.f16 fh, h;\n\tcvt.rn.bf16x2.f32 %0, fh, fl;\n}"
      : "=r"(r) : "r"(v));
  return r;
}
// f16x2 pre-activations x -> bf16x2 GELU(x)
__device__ __forceinline__ uint32_t gelu_f16x2_bf16x2(uint32_t x) {
  const uint32_t c0 = 0x3A623A62u;  // f16(0.7978846) x2
  const uint32_t c1 = 0x28912891u;  // f16(0.0356774) x2
  const uint32_t hf = 0x38003800u;  // 0.5 x2
  uint32_t xx, t, u, th, hx, r;
  asm("mul.rn.f16x2 %0, %1, %1;" : "=r"(xx) : "r"(x));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(t) : "r"(xx), "r"(c1), "r"(c0));
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(u) : "r"(t), "r"(x));
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(th) : "r"(u));
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(hx) : "r"(x), "r"(hf));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(hx), "r"(th), "r"(hx));
  return f16x2_to_bf16x2(r);
}
// The same GELU applied to y = x/2 (the layer-1 weights and b1 are stored halved, exact in
// bf16): x (c0 + c1 x^2) = y (2 c0 + 8 c1 y^2) and 0.5 x (1 + t) = y + y t, one multiply fewer.
__device__ __forceinline__ uint32_t gelu_half_f16x2_bf16x2(uint32_t y) {
  const uint32_t c0 = 0x3E623E62u;  // f16(2 * 0.7978846) x2
  const uint32_t c1 = 0x34913491u;  // f16(8 * 0.0356774) x2
  uint32_t yy, t, u, th, r;
  asm("mul.rn.f16x2 %0, %1, %1;" : "=r"(yy) : "r"(y));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(t) : "r"(yy), "r"(c1), "r"(c0));
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(u) : "r"(t), "r"(y));
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(th) : "r"(u));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(y), "r"(th), "r"(y));
  return f16x2_to_bf16x2(r);
}
// fp32 GELU (same tanh form, MUFU tanh.approx.f32): used where the activation
// feeds an fp32 reduction directly (layer 3 -> the folded layer-4 dot)
__device__ __forceinline__ float gelu_f32(float x) {
  float t;
  const float u = x * fmaf(0.0356774081f, x * x, 0.7978845608f);
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  const float hx = 0.5f * x;
  return fmaf(hx, t, hx);
}
// erf-form GELU in fp32 (the oracle's form, R5) for the TF32 precision mode: GELU(x) = x Phi(x) with
// Phi from erfc(|x|/sqrt 2) by Abramowitz & Stegun 7.1.26, erfc(t) = (a1 k + .. + a5 k^5) e^(-t^2),
// k = 1 / (1 + p t): absolute error <= 2.1e-7 on GELU, 4.2e-7 with the fp32 rounding (2e6-point grid on [-10, 10]
// against scipy's erf), 2500x below the tf32 rounding of a unit activation.  Two MUFU ops (rcp, ex2)
// and 9 FMA-pipe operations instead of erff's ~25 instructions with both branches selected: the
// layer-1 GELU of the TF32 path was issue-bound on erff.
__device__ __forceinline__ float gelu_erf_f32(float x) {
  const float t = fabsf(x) * 0.7071067811865476f;
  float k, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(k) : "f"(fmaf(0.3275911f, t, 1.0f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * t * t));
  const float poly = k * fmaf(k, fmaf(k, fmaf(k, fmaf(k, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f),
                              0.254829592f);
  const float half = 0.5f * poly * e;  // = Phi(-|x|)
  return x * (x >= 0.f ? 1.0f - half : half);
}
// round-to-nearest fp32 -> tf32 (the value the tensor core multiplies; low 13 mantissa bits zero)
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// element-type traits of the MLP GEMMs: bf16 (kind::f16, K16 atoms) or tf32 (kind::tf32, K8 atoms);
// one MMA K atom is 32 bytes of a K-major operand row in both cases
template <bool TF32>
struct Elem {
  static constexpr int BYTES = TF32 ? 4 : 2;
  static constexpr int KATOM = TF32 ? 8 : 16;
  static constexpr uint32_t FMT = TF32 ? 2u : 1u;  // instruction-descriptor a/b format
};
// precision modes of the MLP GEMMs (rc_mlp_desc.precision): 0 bf16, 1 tf32, 2 tf32x3
// (fp32-accurate: a_hi b_hi + a_lo b_hi + a_hi b_lo with tf32 hi/lo operand pairs)
template <int PREC>
struct Prec {
  static constexpr bool TF32 = PREC != 0;
  static constexpr bool X3 = PREC == 2;
  static constexpr int NOP = X3 ? 2 : 1;  // operand copies per tile (hi, lo)
};

template <bool TF32>
__device__ __forceinline__ void mma_cta(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (TF32) rcx::mma_tf32(d, a, b, idesc, acc); else rcx::mma_bf16(d, a, b, idesc, acc);
}
template <bool TF32>
__device__ __forceinline__ void mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (TF32) rcx::mma_tf32_pair(d, a, b, idesc, acc); else rcx::mma_bf16_pair(d, a, b, idesc, acc);
}

__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// UMMA K-major descriptor for a 32/64/128-byte swizzled tile (8-row atoms, SBO = 8 rows)
template <int ROW_BYTES>
__device__ __forceinline__ uint64_t desc_sw(const void *smem) {
  constexpr uint64_t layout = ROW_BYTES == 128 ? 2 : ROW_BYTES == 64 ? 4 : 6;
  uint64_t d = (uint64_t)((rcx::smem_u32(smem) & 0x3FFFF) >> 4);
  d |= (uint64_t)((8 * ROW_BYTES) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(rcx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read3() { asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// named barrier over the first `n` threads of the CTA (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void bar_sync_1(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// 16 bf16 columns (32 B) of row `row` into a [rows][64] bf16 staging block laid out
// as the TMA 128-byte swizzle expects (16-byte unit u of row r at r*128 + ((u ^ r%8) * 16));
// `unit0` = the even 16-byte unit (0, 2, 4, 6) the 16 columns start at.
__device__ __forceinline__ void stage_sw128(uint8_t *blk, int row, int unit0, const uint32_t (&pk)[8]) {
  uint8_t *r = blk + row * 128;
  const int x = row & 7;
  *reinterpret_cast<uint4 *>(r + ((unit0 ^ x) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  *reinterpret_cast<uint4 *>(r + (((unit0 + 1) ^ x) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
}

}  // namespace rcm
