// peer.cuh — fused cross-GPU combine over NVLink peer memory.
// Included by reduce.cu after the tree helpers.
//
// The CTA that has just built this rank's root pair (last-leaf retire, TMA
// last CTA, or the PDL tree kernel) finishes the job for the whole job:
//   1. thread r < G stores the root into peer r's symmetric buffer, slot
//      [epoch & 1][rank] (plain NVLink stores, then fence.sc.sys), and sets
//      peer r's flag [rank] = epoch with st.release.sys;
//   2. thread t < G waits (ld.acquire.sys, bounded spin) until this rank's
//      flag [t] >= epoch, i.e. rank t's pair for this epoch has landed here;
//   3. the CTA runs the same balanced tree as tf_merge_tree over the G pairs
//      of slot [epoch & 1] and writes the global (value, error).
// Every rank computes the identical tree over identical bytes, so all ranks
// hold bit-identical results — the NCCL all-gather + merge kernel, fused
// into the reduction's last step.  Epoch parity double-buffers the slots: a
// rank can only reuse parity p two calls later, after every peer has already
// consumed it (completing call k+1 needs every peer's k+1 publication, which
// each peer issues only after it finished reading call k).  A wait that
// exceeds timeout_ns (%globaltimer) stamps error[0] = epoch, ORs the missing
// ranks into error[1] and yields NaN for THAT call only (the stamp is per
// epoch, never sticky): the host (dist.py) raises RuntimeError on it, and
// since the late rank's own peers then time out on it in turn, every rank of
// the group fails the same call instead of some ranks hanging.

namespace tfb {

constexpr int kMaxPeers = 16;

struct PeerCtx {
  int32_t world;                  // G <= kMaxPeers
  int32_t rank;
  int32_t* error;                 // local device words: [0] epoch of the last timed-out call,
                                  // [1] bitmask of the ranks that call never heard from
  void* bufs[kMaxPeers];          // peer r's pair buffer: [2][G] Pair<A>
  uint32_t* flags[kMaxPeers];     // peer r's flags: [G] uint32 (epoch of rank g's last publication)
  unsigned long long timeout_ns;  // bound of the wait (device %globaltimer nanoseconds)
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Out of line: the combine runs once per launch and must not widen the hot
// loop's register allocation (inlined, it cost leaves_kernel 14 registers and
// one CTA per SM).
template <int M, typename A, int BAR, int NT>
__device__ __noinline__ void peer_finish(Pair<A> root, Pair<A>* out, const PeerCtx* peer, uint32_t epoch,
                                         Pair<A>* smem) {
  const int t = threadIdx.x;
  group_sync<BAR, NT>();
  if (t == 0) smem[0] = root;
  group_sync<BAR, NT>();
  const Pair<A> mine = smem[0];
  group_sync<BAR, NT>();
  const int G = peer->world;
  const int rank = peer->rank;
  const int parity = static_cast<int>(epoch & 1u);
  if (t < G) {
    Pair<A>* dst = static_cast<Pair<A>*>(peer->bufs[t]) + parity * G + rank;
    volatile A* d = reinterpret_cast<volatile A*>(dst);
    d[0] = mine.s;
    d[1] = mine.e;
    __threadfence_system();
    st_release_sys(peer->flags[t] + rank, epoch);
  }
  __shared__ int missing;
  if (t == 0) missing = 0;
  group_sync<BAR, NT>();
  if (t < G) {
    const uint32_t* f = peer->flags[rank] + t;
    const unsigned long long t0 = global_ns();
    while (static_cast<int32_t>(ld_acquire_sys(f) - epoch) < 0) {
      if (global_ns() - t0 > peer->timeout_ns) {
        atomicOr(&missing, 1 << t);
        break;
      }
      __nanosleep(256);
    }
  }
  group_sync<BAR, NT>();
  Pair<A> global = tree_over<M, A, NT, BAR>(static_cast<const Pair<A>*>(peer->bufs[rank]) + parity * G, G, smem);
  if (t == 0) {
    if (missing) {  // a peer never arrived: poison this call instead of a silent partial sum
      peer->error[1] = missing;
      __threadfence();
      peer->error[0] = static_cast<int32_t>(epoch);
      global.s = A(__longlong_as_double(0x7FF8000000000000ll));
      global.e = global.s;
    }
    *out = global;
  }
}

// All NT threads of the group call this; `root` is valid in thread 0.
template <int M, typename A, int BAR = 0, int NT = kThreads>
__device__ __forceinline__ void finish_root(Pair<A> root, Pair<A>* out, const PeerCtx* peer, uint32_t epoch,
                                            Pair<A>* smem) {
  if (peer == nullptr) {
    if (threadIdx.x == 0) *out = root;
    return;
  }
  peer_finish<M, A, BAR, NT>(root, out, peer, epoch, smem);
}

}  // namespace tfb
