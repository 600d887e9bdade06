// alu_probe.cu -- issue throughput of the epilogue's candidate instructions on sm_100a.
// Each kernel runs `iters` rounds of 16 independent chains of one instruction on W warps per SM (one
// CTA per SM) and reports cycles per warp-instruction per SM sub-partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_probe tools/alu_probe.cu
#include <cstdint>
#include <cstdio>

template <int OP>
__global__ void k(uint32_t* out, int iters, float t) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 977u + i * 131u;
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (OP == 0) {  // FADD2
        asm volatile("{\n\t.reg .b64 ra, rc, rd;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rc, {%2, %2};\n\t"
                     "add.rn.f32x2 rd, ra, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                     : "+r"(r[i]), "+r"(r[i + 1]) : "f"(t));
      } else if (OP == 1) {  // I2IP (cvt.pack.sat.u8.s32)
        asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(r[i]) : "r"(r[i + 1]));
        asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(r[i + 1]) : "r"(r[i]));
      } else if (OP == 2) {  // PRMT
        asm volatile("prmt.b32 %0, %0, %1, 0x4602;" : "+r"(r[i]) : "r"(r[i + 1]));
        asm volatile("prmt.b32 %0, %0, %1, 0x4602;" : "+r"(r[i + 1]) : "r"(r[i]));
      } else if (OP == 3) {  // FFMA.SAT with an immediate
        float a = __uint_as_float(r[i]), b = __uint_as_float(r[i + 1]);
        asm volatile("fma.rn.sat.f32 %0, %0, 0f46000000, %1;" : "+f"(a) : "f"(t));
        asm volatile("fma.rn.sat.f32 %0, %0, 0f46000000, %1;" : "+f"(b) : "f"(t));
        r[i] = __float_as_uint(a); r[i + 1] = __float_as_uint(b);
      } else if (OP == 4) {  // F2FP (cvt.rn.f16x2.f32)
        float a = __uint_as_float(r[i]), b = __uint_as_float(r[i + 1]);
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r[i]) : "f"(a), "f"(b));
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r[i + 1]) : "f"(b), "f"(a));
      } else if (OP == 5) {  // FSET (set.gt.u32.f32: 0xFFFFFFFF / 0)
        asm volatile("set.gt.u32.f32 %0, %1, %2;" : "=r"(r[i]) : "f"(__uint_as_float(r[i])), "f"(t));
        asm volatile("set.gt.u32.f32 %0, %1, %2;" : "=r"(r[i + 1]) : "f"(__uint_as_float(r[i + 1])), "f"(t));
      } else if (OP == 6) {  // IADD3
        asm volatile("add.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(r[i + 1]));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(r[i + 1]) : "r"(r[i]));
      } else if (OP == 7) {  // FADD (scalar)
        float a = __uint_as_float(r[i]), b = __uint_as_float(r[i + 1]);
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a) : "f"(t));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(b) : "f"(t));
        r[i] = __float_as_uint(a); r[i + 1] = __float_as_uint(b);
      }
    }
  }
  const long long c1 = clock64();
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) x ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1u << 20] = (uint32_t)(c1 - c0);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, (1u << 20) * 4 + 64);
  const char* names[] = {"FADD2 (add.rn.f32x2)", "I2IP (cvt.pack.sat.u8.s32)", "PRMT", "FFMA.SAT imm",
                         "F2FP (cvt.rn.f16x2.f32)", "FSET (set.gt.u32.f32)", "IADD", "FADD"};
  const int iters = 4096;
  for (int W : {4, 8, 16}) {
    for (int op = 0; op < 8; ++op) {
      void (*fn)(uint32_t*, int, float) = nullptr;
      switch (op) {
        case 0: fn = k<0>; break; case 1: fn = k<1>; break; case 2: fn = k<2>; break; case 3: fn = k<3>; break;
        case 4: fn = k<4>; break; case 5: fn = k<5>; break; case 6: fn = k<6>; break; default: fn = k<7>; break;
      }
      fn<<<148, 32 * W>>>(d, iters, 0.5f);
      fn<<<148, 32 * W>>>(d, iters, 0.5f);
      cudaDeviceSynchronize();
      uint32_t cyc;
      cudaMemcpy(&cyc, d + (1u << 20), 4, cudaMemcpyDeviceToHost);
      const double instr_per_warp = (double)iters * 16;          // warp-instructions per warp
      const double per_smsp = instr_per_warp * W / 4;           // per sub-partition
      printf("W=%2d %-28s %.2f cycles per warp-instruction per SMSP\n", W, names[op], cyc / per_smsp);
    }
  }
  return 0;
}
