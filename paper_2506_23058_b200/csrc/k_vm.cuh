// k_vm.cuh -- `map f xs...` for an arbitrary (first-order, scalar) lambda.
//
// The reference applies a Closure per element (oracle.py:274-280, 94-107),
// walking the lambda's AST with a fresh environment each time.  Here the
// host compiles the lambda once into a short register program (vm.py) and
// every GPU thread interprets it for its elements.  The program travels in
// the kernel's parameter space (constant bank), so instruction fetch is a
// uniform broadcast; registers are a per-thread local array.
#pragma once
#include "common.cuh"

namespace ixg {

struct VmProgram {
  ixg_vm_insn insn[IXG_VM_MAX_INSN];
  ixg_array in[IXG_VM_MAX_IN];
  ixg_array out[IXG_VM_MAX_OUT];
  ixg_pred pred[IXG_VM_MAX_PRED];
  int ninsn, nin, nout, npred;
};

IXG_DEV long long vm_load(const ixg_array& a, long long i) {
  switch (a.dt) {
    case IXG_I32: return reinterpret_cast<const int32_t*>(a.ptr)[i];
    case IXG_U8: return reinterpret_cast<const uint8_t*>(a.ptr)[i];
    default: return reinterpret_cast<const long long*>(a.ptr)[i];
  }
}
IXG_DEV void vm_store(const ixg_array& a, long long i, long long v) {
  switch (a.dt) {
    case IXG_I32: reinterpret_cast<int32_t*>(const_cast<void*>(a.ptr))[i] = (int32_t)v; break;
    case IXG_U8: reinterpret_cast<uint8_t*>(const_cast<void*>(a.ptr))[i] = (uint8_t)(v != 0); break;
    default: reinterpret_cast<long long*>(const_cast<void*>(a.ptr))[i] = v; break;
  }
}

__global__ void __launch_bounds__(256) k_map_vm(const __grid_constant__ VmProgram P, long long n, int stmt,
                                               ixg_status* st) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    long long r[IXG_VM_REGS];
    int pc = 0;
    bool failed = false;
    while (pc < P.ninsn) {
      const ixg_vm_insn& I = P.insn[pc++];
      switch (I.op) {
        case IXG_VM_IN: r[I.dst] = vm_load(P.in[I.a], i); break;
        case IXG_VM_CONST: r[I.dst] = I.imm; break;
        case IXG_VM_ADD:
        case IXG_VM_SUB:
        case IXG_VM_MUL: {  // int64, checked: the reference's ints are unbounded (oracle.py:214-240)
          long long v;
          const bool o = I.op == IXG_VM_ADD ? add_ovf(r[I.a], r[I.b], &v)
                         : I.op == IXG_VM_SUB ? sub_ovf(r[I.a], r[I.b], &v)
                                              : mul_ovf(r[I.a], r[I.b], &v);
          if (o) {
            status_overflow(st, stmt, i);
            failed = true;
            pc = P.ninsn;
            break;
          }
          r[I.dst] = v;
          break;
        }
        case IXG_VM_EQ: r[I.dst] = r[I.a] == r[I.b]; break;
        case IXG_VM_NE: r[I.dst] = r[I.a] != r[I.b]; break;
        case IXG_VM_LT: r[I.dst] = r[I.a] < r[I.b]; break;
        case IXG_VM_LE: r[I.dst] = r[I.a] <= r[I.b]; break;
        case IXG_VM_GT: r[I.dst] = r[I.a] > r[I.b]; break;
        case IXG_VM_GE: r[I.dst] = r[I.a] >= r[I.b]; break;
        case IXG_VM_NOT: r[I.dst] = r[I.a] == 0; break;
        case IXG_VM_MOV: r[I.dst] = r[I.a]; break;
        case IXG_VM_JZ:
          if (r[I.a] == 0) pc = I.c;
          break;
        case IXG_VM_JMP: pc = I.c; break;
        case IXG_VM_IDX: {
          const long long k = r[I.a];
          const ixg_array& A = P.in[I.b];
          if ((unsigned long long)k >= (unsigned long long)A.len) {
            if (I.imm) {
              status_fail(st, IXG_OOB, stmt, i, I.c);
              failed = true;
              pc = P.ninsn;
              break;
            }
          }
          r[I.dst] = vm_load(A, k);
          break;
        }
        case IXG_VM_PRED: r[I.dst] = pred_eval(P.pred[I.b], r[I.a]); break;
        case IXG_VM_OUT: vm_store(P.out[I.b], i, r[I.a]); break;
        case IXG_VM_LEN: r[I.dst] = P.in[I.b].len; break;
        default: pc = P.ninsn; break;
      }
    }
    (void)failed;
  }
}

}  // namespace ixg
