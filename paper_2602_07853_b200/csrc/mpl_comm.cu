// mpl_comm.cu — the slab decomposition across GPUs.
//
// Rank r owns the 4-cell blocks [X_r, X_{r+1}) along x: their quadrature points (cells), the
// particles whose base cell lies there, and the nodes those cells touch.  The node plane x = 4 X_{r+1}
// is shared with rank r+1; both ranks keep identical values on it:
//   * C2N, gradient, Jacobi diagonal and every HVP produce partial sums on the shared planes, which
//     are completed by one neighbour exchange (halo_sum_nodes: dense y-z plane buffers, send both
//     ways, add); additions are commutative, so both copies are bitwise equal and every later update
//     of a shared node (PCG x, r, p; Newton v) stays identical on the two ranks;
//   * dot products and the energy count a shared node once (owner flag: the upper rank owns the
//     plane unless it does not hold the node), and are summed over ranks by allreduce (fp64);
//   * P2Q of the first cell plane of a slab needs the particles of the last cell plane of the lower
//     slab: those are copied in as ghosts (pid < 0) every step (redistribute_particles);
//   * G2P of particles in the last cell plane needs the velocity of the next slab's second node plane
//     (ghost_nodes_from_upper).
// Transport: NCCL (ncclAllReduce, grouped ncclSend/ncclRecv, loaded with dlopen so the library does not
// link NCCL) when every rank is its own process, or an in-process loopback group when the ranks are host
// threads of one process (used to test the decomposition on one GPU: each collective synchronises the
// rank's stream, meets the other threads at a host barrier and copies/reduces with ordinary kernels —
// no kernel ever waits on another rank's kernel).
#include <dlfcn.h>
#include <nccl.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mpl_common.cuh"

// =============================================================================================
// loopback group
// =============================================================================================
struct mpl_group_s {
    int R = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    bool broken = false;
    std::vector<const void *> pa, pb;
    std::vector<size_t> sa, sb;
};

namespace {

constexpr int MAX_LOOPBACK = 64;

// MPL_LOOPBACK_SERIAL=1 (debugging aid): library calls of different ranks never run at the same time.
// Every C-ABI entry holds a process-wide recursive lock (ApiLock); a rank waiting at a loopback barrier
// releases it (all recursion levels) and re-acquires it afterwards.  With CUDA_LAUNCH_BLOCKING=1 a
// device fault is then reported by the rank whose kernel caused it.
bool group_barrier_impl(mpl_group g);
bool group_barrier(mpl_group g) {
    if (!serial_mode()) return group_barrier_impl(g);
    const int depth = api_lock_release_all();
    bool ok = group_barrier_impl(g);
    api_lock_reacquire(depth);
    return ok;
}

bool group_barrier_impl(mpl_group g) {
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->broken) return false;
    const long my = g->gen;
    if (++g->arrived == g->R) {
        g->arrived = 0;
        g->gen++;
        g->cv.notify_all();
        return true;
    }
    static const int timeout_s = [] {
        const char *e = getenv("MPL_LOOPBACK_TIMEOUT");
        return e ? atoi(e) : 300;
    }();
    if (!g->cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return g->gen != my || g->broken; }) ||
        g->broken) {
        g->broken = true;  // a rank failed or never arrived: release everyone with an error
        g->cv.notify_all();
        return false;
    }
    return true;
}

struct PtrList {
    const double *p[MAX_LOOPBACK];
};
__global__ void k_sum_ranks(int R, int64_t n, PtrList l, double *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < R; q++) s += l.p[q][i];  // fixed order: identical on every rank
        out[i] = s;
    }
}

struct LoopbackComm : Comm {
    mpl_group g;
    DevBuf tmp;
    ~LoopbackComm() override {
        if (tmp.p) cudaFree(tmp.p);
    }
    mpl_status fail(mpl_ctx ctx, const char *what) {
        ctx->err = std::string("loopback group: ") + what + " (a rank failed or did not arrive)";
        return MPL_ERR_NCCL;
    }
    mpl_status allreduce(mpl_ctx ctx, double *dev, int64_t n) override {
        if (n <= 0) return MPL_OK;
        MPL_CHECK(ensure(ctx, tmp, (size_t)n * 8));
        MPL_CUDA(cudaStreamSynchronize(ctx->stream));
        g->pa[rank] = dev;
        if (!group_barrier(g)) return fail(ctx, "allreduce");
        PtrList l;
        for (int q = 0; q < nranks; q++) l.p[q] = (const double *)g->pa[q];
        k_sum_ranks<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, ctx->stream>>>(nranks, n, l,
                                                                                               (double *)tmp.p);
        MPL_CUDA(cudaGetLastError());
        MPL_CUDA(cudaStreamSynchronize(ctx->stream));
        if (!group_barrier(g)) return fail(ctx, "allreduce");  // every rank has read every partial
        MPL_CUDA(cudaMemcpyAsync(dev, tmp.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        return MPL_OK;
    }
    mpl_status neighbors(mpl_ctx ctx, const void *send_lo, size_t n_send_lo, void *recv_lo, size_t n_recv_lo,
                         const void *send_hi, size_t n_send_hi, void *recv_hi, size_t n_recv_hi) override {
        MPL_CUDA(cudaStreamSynchronize(ctx->stream));
        g->pa[rank] = rank > 0 ? send_lo : nullptr;
        g->sa[rank] = rank > 0 ? n_send_lo : 0;
        g->pb[rank] = rank < nranks - 1 ? send_hi : nullptr;
        g->sb[rank] = rank < nranks - 1 ? n_send_hi : 0;
        if (!group_barrier(g)) return fail(ctx, "neighbour exchange");
        mpl_status st = MPL_OK;
        if (rank > 0 && n_recv_lo) {  // from rank-1's send_hi
            if (g->sb[rank - 1] != n_recv_lo) st = MPL_ERR_INVALID_ARG;
            else if (cudaMemcpyAsync(recv_lo, g->pb[rank - 1], n_recv_lo, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
                st = MPL_ERR_CUDA;
        }
        if (rank < nranks - 1 && n_recv_hi) {  // from rank+1's send_lo
            if (g->sa[rank + 1] != n_recv_hi) st = MPL_ERR_INVALID_ARG;
            else if (cudaMemcpyAsync(recv_hi, g->pa[rank + 1], n_recv_hi, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
                st = MPL_ERR_CUDA;
        }
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess && st == MPL_OK) st = MPL_ERR_CUDA;
        if (!group_barrier(g)) return fail(ctx, "neighbour exchange");
        if (st != MPL_OK) ctx->err = "loopback neighbour exchange: size mismatch or copy failure";
        return st;
    }
};

// =============================================================================================
// NCCL (dlopen'ed: the library itself does not link libnccl)
// =============================================================================================
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (tried) return api;
    tried = true;
    // prefer an NCCL already loaded in the process (torch's), else the system one
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
        return api;
    }
#define SYM(field, name)                                                   \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));     \
    if (!api.field) {                                                      \
        api.why = std::string("libnccl.so.2 lacks ") + name;               \
        return api;                                                        \
    }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(AllReduce, "ncclAllReduce");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.ok = true;
    return api;
}

#define NCCL_CHECK(call)                                                                        \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess) {                                                                \
            ctx->err = std::string("NCCL error: ") + nccl().GetErrorString(r_) + " at " +       \
                       __FILE__ + ":" + std::to_string(__LINE__);                               \
            return MPL_ERR_NCCL;                                                                \
        }                                                                                       \
    } while (0)

struct NcclComm : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) nccl().CommDestroy(comm);
    }
    mpl_status allreduce(mpl_ctx ctx, double *dev, int64_t n) override {
        if (n <= 0) return MPL_OK;
        NCCL_CHECK(nccl().AllReduce(dev, dev, (size_t)n, ncclFloat64, ncclSum, comm, ctx->stream));
        return MPL_OK;
    }
    mpl_status neighbors(mpl_ctx ctx, const void *send_lo, size_t n_send_lo, void *recv_lo, size_t n_recv_lo,
                         const void *send_hi, size_t n_send_hi, void *recv_hi, size_t n_recv_hi) override {
        NCCL_CHECK(nccl().GroupStart());
        if (rank > 0) {
            if (n_send_lo) NCCL_CHECK(nccl().Send(send_lo, n_send_lo, ncclUint8, rank - 1, comm, ctx->stream));
            if (n_recv_lo) NCCL_CHECK(nccl().Recv(recv_lo, n_recv_lo, ncclUint8, rank - 1, comm, ctx->stream));
        }
        if (rank < nranks - 1) {
            if (n_send_hi) NCCL_CHECK(nccl().Send(send_hi, n_send_hi, ncclUint8, rank + 1, comm, ctx->stream));
            if (n_recv_hi) NCCL_CHECK(nccl().Recv(recv_hi, n_recv_hi, ncclUint8, rank + 1, comm, ctx->stream));
        }
        NCCL_CHECK(nccl().GroupEnd());
        return MPL_OK;
    }
};

// =============================================================================================
// interface-plane kernels
// =============================================================================================
__device__ __forceinline__ int local_id(int lx, int ly, int lz) { return (lx * 4 + ly) * 4 + lz; }

__global__ void k_interface_lists(int T_, const int *__restrict__ coord, int xlo, int xhi, int *lo_list, int *hi_list,
                                  int *counts) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T_) return;
    const int bx = coord[3 * t];
    if (bx == xlo) lo_list[atomicAdd(&counts[0], 1)] = t;
    if (bx == xhi) hi_list[atomicAdd(&counts[1], 1)] = t;
}

// Compact face messages: entry k of a (sorted) face list carries the 16 nodes (ly, lz) of the tile's
// node plane lx, nv vectors each, at dst[(16 k + 4 ly + lz) nv + v].
template <class T>
__global__ void k_face_pack(const int *__restrict__ list, int lx, int nv, const vec4<T> *__restrict__ a,
                            const vec4<T> *__restrict__ b, vec4<T> *__restrict__ dst) {
    const int t = list[blockIdx.x];
    const int ly = threadIdx.x >> 2, lz = threadIdx.x & 3;
    const int64_t n = (int64_t)t * 64 + local_id(lx, ly, lz);
    const int64_t q = ((int64_t)blockIdx.x * 16 + threadIdx.x) * nv;
    dst[q] = a[n];
    if (nv > 1) dst[q + 1] = b[n];
}

// received entry k (the neighbour's k-th face tile) -> local tile map[k] (-1: not held here, the
// neighbour's partial is then complete on its own); MODE 0: add (sum of partials), MODE 1: set (ghost)
template <class T, int MODE>
__global__ void k_face_unpack(const int *__restrict__ map, int lx, int nv, const vec4<T> *__restrict__ src,
                              vec4<T> *__restrict__ a, vec4<T> *__restrict__ b) {
    const int t = map[blockIdx.x];
    if (t < 0) return;
    const int ly = threadIdx.x >> 2, lz = threadIdx.x & 3;
    const int64_t n = (int64_t)t * 64 + local_id(lx, ly, lz);
    const int64_t q = ((int64_t)blockIdx.x * 16 + threadIdx.x) * nv;
    const vec4<T> s = src[q];
    if (MODE == 0) {
        vec4<T> x = a[n];
        x.x += s.x; x.y += s.y; x.z += s.z; x.w += s.w;
        a[n] = x;
        if (nv > 1) {
            const vec4<T> s2 = src[q + 1];
            vec4<T> y = b[n];
            y.x += s2.x; y.y += s2.y; y.z += s2.z; y.w += s2.w;
            b[n] = y;
        }
    } else {
        a[n] = s;
    }
}

// C2N halo: (mv, m) partials of plane lx = 0; a tile the upper neighbour holds makes it the owner of
// the shared nodes (this rank's copy is then not counted in dots / energy)
template <class T>
__global__ void k_c2n_face_unpack(const int *__restrict__ map, int upper, const vec4<T> *__restrict__ src,
                                  vec4<T> *__restrict__ mvm, uint8_t *__restrict__ own) {
    const int t = map[blockIdx.x];
    if (t < 0) return;
    const int ly = threadIdx.x >> 2, lz = threadIdx.x & 3;
    const int64_t n = (int64_t)t * 64 + local_id(0, ly, lz);
    const vec4<T> s = src[(int64_t)blockIdx.x * 16 + threadIdx.x];
    vec4<T> x = mvm[n];
    x.x += s.x; x.y += s.y; x.z += s.z; x.w += s.w;
    mvm[n] = x;
    if (upper) own[n] = 0;
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// =============================================================================================
// particle redistribution (migration to the neighbour slabs + ghost copies)
// =============================================================================================
// record: 25 reals (x 3, v 3, F 9, G 9, vol) then int32 mat, int32 pid
template <class T> constexpr int rec_bytes() { return (int)((25 * sizeof(T) + 8 + 15) / 16 * 16); }

template <class T>
__device__ __forceinline__ int base_x(const GridP &g, T x) {
    return (int)floor((x - T(g.origin[0])) * T(g.inv_dx) - T(0.5));
}

// code: 0 keep, 1 -> lower neighbour, 2 -> upper neighbour, 3 drop (ghost); out-of-range -> error
template <class T>
__global__ void k_classify(GridP g, int64_t n, const T *__restrict__ x, const int *__restrict__ pid, int A_lo, int A,
                           int B, int B_hi, int *__restrict__ code, unsigned long long *__restrict__ cnt, int *bad) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int c;
    if (pid[p] < 0) {
        c = 3;
    } else {
        const int bx = base_x<T>(g, x[3 * p]);
        if (bx >= A && bx < B) c = 0;
        else if (bx >= A_lo && bx < A) c = 1;
        else if (bx >= B && bx < B_hi) c = 2;
        else {
            c = 3;
            atomicMin(bad, pid[p]);
        }
    }
    code[p] = c;
    atomicAdd(&cnt[c], 1ull);
}

template <class T>
__device__ __forceinline__ void write_rec(char *r, int64_t p, const T *x, const T *v, const T *F, const T *G,
                                          const T *vol, const int *mat, const int *pid, int pid_override, bool use_ov) {
    T *q = reinterpret_cast<T *>(r);
#pragma unroll
    for (int a = 0; a < 3; a++) { q[a] = x[3 * p + a]; q[3 + a] = v[3 * p + a]; }
#pragma unroll
    for (int a = 0; a < 9; a++) { q[6 + a] = F[9 * p + a]; q[15 + a] = G[9 * p + a]; }
    q[24] = vol[p];
    int *iq = reinterpret_cast<int *>(r + 25 * sizeof(T));
    iq[0] = mat[p];
    iq[1] = use_ov ? pid_override : pid[p];
}

struct PartOut {
    void *x, *v, *F, *G, *vol;
    int *mat, *pid;
};

// kept particles -> new arrays at atomic offsets; leavers -> send records
template <class T>
__global__ void k_migrate_pack(int64_t n, const int *__restrict__ code, const T *__restrict__ x, const T *__restrict__ v,
                               const T *__restrict__ F, const T *__restrict__ G, const T *__restrict__ vol,
                               const int *__restrict__ mat, const int *__restrict__ pid, PartOut o, char *send_lo,
                               char *send_hi, unsigned long long *cursor) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int c = code[p];
    if (c == 3) return;
    const int64_t k = (int64_t)atomicAdd(&cursor[c], 1ull);
    if (c == 0) {
        T *xo = (T *)o.x, *vo = (T *)o.v, *Fo = (T *)o.F, *Go = (T *)o.G, *vlo = (T *)o.vol;
#pragma unroll
        for (int a = 0; a < 3; a++) { xo[3 * k + a] = x[3 * p + a]; vo[3 * k + a] = v[3 * p + a]; }
#pragma unroll
        for (int a = 0; a < 9; a++) { Fo[9 * k + a] = F[9 * p + a]; Go[9 * k + a] = G[9 * p + a]; }
        vlo[k] = vol[p];
        o.mat[k] = mat[p];
        o.pid[k] = pid[p];
    } else {
        char *dst = (c == 1 ? send_lo : send_hi) + k * rec_bytes<T>();
        write_rec<T>(dst, p, x, v, F, G, vol, mat, pid, 0, false);
    }
}

// append records at offset `at`; ghost: store pid as ~pid (negative)
template <class T>
__global__ void k_unpack_recs(int64_t m, const char *__restrict__ recs, int64_t at, int ghost, PartOut o) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const char *r = recs + i * rec_bytes<T>();
    const T *q = reinterpret_cast<const T *>(r);
    const int *iq = reinterpret_cast<const int *>(r + 25 * sizeof(T));
    const int64_t k = at + i;
    T *xo = (T *)o.x, *vo = (T *)o.v, *Fo = (T *)o.F, *Go = (T *)o.G, *vlo = (T *)o.vol;
#pragma unroll
    for (int a = 0; a < 3; a++) { xo[3 * k + a] = q[a]; vo[3 * k + a] = q[3 + a]; }
#pragma unroll
    for (int a = 0; a < 9; a++) { Fo[9 * k + a] = q[6 + a]; Go[9 * k + a] = q[15 + a]; }
    vlo[k] = q[24];
    o.mat[k] = iq[0];
    o.pid[k] = ghost ? ~iq[1] : iq[1];
}

// owned particles of the last cell plane of the slab -> ghost records for the upper neighbour
template <class T>
__global__ void k_ghost_pack(GridP g, int64_t n, int plane, const T *__restrict__ x, const T *__restrict__ v,
                             const T *__restrict__ F, const T *__restrict__ G, const T *__restrict__ vol,
                             const int *__restrict__ mat, const int *__restrict__ pid, char *send,
                             unsigned long long *cursor) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (base_x<T>(g, x[3 * p]) != plane) return;
    const int64_t k = (int64_t)atomicAdd(cursor, 1ull);
    write_rec<T>(send + k * rec_bytes<T>(), p, x, v, F, G, vol, mat, pid, 0, false);
}

template <class T>
__global__ void k_count_plane(GridP g, int64_t n, int plane, const T *__restrict__ x, unsigned long long *cnt) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (base_x<T>(g, x[3 * p]) == plane) atomicAdd(cnt, 1ull);
}

// ---- owned-particle export in ascending id order --------------------------------------------
__global__ void k_owned_keys(int64_t n, const int *__restrict__ pid, int *__restrict__ keys, int *__restrict__ idx,
                             unsigned long long *cnt) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (pid[p] < 0) return;
    const int64_t k = (int64_t)atomicAdd(cnt, 1ull);
    keys[k] = pid[p];
    idx[k] = (int)p;
}

template <class T>
__global__ void k_gather_rows(int64_t m, int w, const int *__restrict__ idx, const T *__restrict__ in, T *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m * w) return;
    const int64_t r = i / w;
    const int a = (int)(i % w);
    out[i] = in[(int64_t)idx[r] * w + a];
}

__global__ void k_base_rows(int64_t m, const int *__restrict__ idx, const int *__restrict__ skey,
                            const int *__restrict__ coord, int32_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int key = skey[idx[i]], t = key >> 6, l = key & 63;
    out[3 * i + 0] = coord[3 * t] * 4 + (l >> 4);
    out[3 * i + 1] = coord[3 * t + 1] * 4 + ((l >> 2) & 3);
    out[3 * i + 2] = coord[3 * t + 2] * 4 + (l & 3);
}

}  // namespace

// =============================================================================================
// host side
// =============================================================================================
mpl_status comm_create(mpl_ctx ctx, const mpl_config *cfg) {
    if (cfg->nranks <= 1) return MPL_OK;
    if (cfg->rank < 0 || cfg->rank >= cfg->nranks) return MPL_ERR_INVALID_ARG;
    if (cfg->loopback) {
        mpl_group g = cfg->loopback;
        if (g->R != cfg->nranks || cfg->nranks > MAX_LOOPBACK) return MPL_ERR_INVALID_ARG;
        LoopbackComm *c = new LoopbackComm();
        c->g = g;
        c->rank = cfg->rank;
        c->nranks = cfg->nranks;
        ctx->comm = c;
        return MPL_OK;
    }
    if (!cfg->nccl_unique_id) {
        ctx->err = "nranks > 1 needs nccl_unique_id (from mpl_nccl_unique_id on rank 0) or a loopback group";
        return MPL_ERR_INVALID_ARG;
    }
    NcclApi &api = nccl();
    if (!api.ok) {
        ctx->err = api.why;
        return MPL_ERR_NCCL;
    }
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, sizeof id);
    NcclComm *c = new NcclComm();
    c->rank = cfg->rank;
    c->nranks = cfg->nranks;
    ncclResult_t r = api.CommInitRank(&c->comm, cfg->nranks, id, cfg->rank);
    if (r != ncclSuccess) {
        ctx->err = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
        c->comm = nullptr;
        delete c;
        return MPL_ERR_NCCL;
    }
    ctx->comm = c;
    return MPL_OK;
}

void comm_destroy(mpl_ctx ctx) {
    delete ctx->comm;
    ctx->comm = nullptr;
}

mpl_status allreduce_d(mpl_ctx ctx, double *dev, int64_t n) {
    if (!multi(ctx)) return MPL_OK;
    return ctx->comm->allreduce(ctx, dev, n);
}

// Collective error agreement: every rank returns an error if any rank failed (a rank that returned
// early would otherwise leave the others waiting in the next collective).
mpl_status agree(mpl_ctx ctx, mpl_status local) {
    if (!multi(ctx)) return local;
    double *d = (double *)((char *)ctx->scalars.p + 3072);
    double h = local != MPL_OK ? 1.0 : 0.0;
    MPL_CUDA(cudaMemcpyAsync(d, &h, 8, cudaMemcpyHostToDevice, ctx->stream));
    MPL_CHECK(ctx->comm->allreduce(ctx, d, 1));
    MPL_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
    MPL_CUDA(cudaStreamSynchronize(ctx->stream));
    if (local != MPL_OK) return local;
    if (h > 0.0) {
        ctx->err = "another slab rank failed in this collective call";
        return MPL_ERR_STATE;
    }
    return MPL_OK;
}

// debug build: the tile tables are self-consistent (neighbour indices < T, coords in range)
mpl_status debug_check_tiles(mpl_ctx ctx, const char *where) {
    const int T_ = ctx->T;
    MPL_CUDA(cudaStreamSynchronize(ctx->stream));
    std::vector<int> np_(8 * (size_t)T_), nm(8 * (size_t)T_), co(3 * (size_t)T_);
    if (T_) {
        MPL_CUDA(cudaMemcpy(np_.data(), ctx->t_nplus.p, np_.size() * 4, cudaMemcpyDeviceToHost));
        MPL_CUDA(cudaMemcpy(nm.data(), ctx->t_nminus.p, nm.size() * 4, cudaMemcpyDeviceToHost));
        MPL_CUDA(cudaMemcpy(co.data(), ctx->t_coord.p, co.size() * 4, cudaMemcpyDeviceToHost));
    }
    for (int t = 0; t < T_; t++)
        for (int o = 0; o < 8; o++)
            if (np_[8 * t + o] >= T_ || nm[8 * t + o] >= T_ || np_[8 * t + o] < -1) {
                ctx->err = std::string("debug (") + where + "): rank " + std::to_string(ctx->rank) + " tile " +
                           std::to_string(t) + " slot " + std::to_string(o) + " nplus " +
                           std::to_string(np_[8 * t + o]) + " nminus " + std::to_string(nm[8 * t + o]) + " T " +
                           std::to_string(T_) + " coord " + std::to_string(co[3 * t]) + "," +
                           std::to_string(co[3 * t + 1]) + "," + std::to_string(co[3 * t + 2]);
                fprintf(stderr, "%s\n", ctx->err.c_str());
                return MPL_ERR_STATE;
            }
    return MPL_OK;
}

namespace {
// exchange one int64 count with each neighbour: returns (from lower, from upper)
mpl_status exchange_counts(mpl_ctx ctx, unsigned long long to_lo, unsigned long long to_hi, unsigned long long *from_lo,
                           unsigned long long *from_hi) {
    MPL_CHECK(ensure(ctx, ctx->mig_cnt, 256));
    unsigned long long h[4] = {to_lo, to_hi, 0, 0};
    unsigned long long *d = (unsigned long long *)ctx->mig_cnt.p + 24;
    MPL_CUDA(cudaMemcpyAsync(d, h, 16, cudaMemcpyHostToDevice, ctx->stream));
    MPL_CUDA(cudaMemsetAsync(d + 2, 0, 16, ctx->stream));
    MPL_CHECK(ctx->comm->neighbors(ctx, d + 0, 8, d + 2, 8, d + 1, 8, d + 3, 8));
    MPL_CUDA(cudaMemcpyAsync(h, d, 32, cudaMemcpyDeviceToHost, ctx->stream));
    MPL_CUDA(cudaStreamSynchronize(ctx->stream));
    *from_lo = ctx->rank > 0 ? h[2] : 0;
    *from_hi = ctx->rank < ctx->nranks - 1 ? h[3] : 0;
    return MPL_OK;
}
}  // namespace

mpl_status build_interface_lists(mpl_ctx ctx) {
    if (!multi(ctx)) return MPL_OK;
    const int T_ = ctx->T;
    cudaStream_t st = ctx->stream;
    MPL_CHECK(ensure(ctx, ctx->t_lo_list, (size_t)T_ * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->t_hi_list, (size_t)T_ * 4 + 16));
    MPL_CHECK(ensure(ctx, ctx->mig_cnt, 256));
    int *cnt = (int *)ctx->mig_cnt.p;
    MPL_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
    if (T_) {
        k_interface_lists<<<nblk(T_, 256), 256, 0, st>>>(T_, (const int *)ctx->t_coord.p, ctx->slab_lo, ctx->slab_hi,
                                                          (int *)ctx->t_lo_list.p, (int *)ctx->t_hi_list.p, cnt);
        ctx->launches++;
    }
    int h[2];
    MPL_CUDA(cudaMemcpyAsync(h, cnt, 8, cudaMemcpyDeviceToHost, st));
    MPL_CUDA(cudaStreamSynchronize(st));
    ctx->n_lo_tiles = h[0];
    ctx->n_hi_tiles = h[1];
    // sort both face lists by (by, bz) on the host (a few thousand tiles), exchange the keys with the
    // neighbours and match the neighbour's entries to local tiles
    std::vector<int> coord((size_t)3 * T_);
    if (T_) MPL_CUDA(cudaMemcpy(coord.data(), ctx->t_coord.p, coord.size() * 4, cudaMemcpyDeviceToHost));
    const int64_t NB2 = ctx->grid.nb[2];
    auto sorted = [&](DevBuf &list, int n, std::vector<int> &tiles, std::vector<int> &keys) -> mpl_status {
        tiles.resize(n);
        if (n) MPL_CUDA(cudaMemcpy(tiles.data(), list.p, (size_t)n * 4, cudaMemcpyDeviceToHost));
        std::sort(tiles.begin(), tiles.end(), [&](int a, int b) {
            return coord[3 * a + 1] * NB2 + coord[3 * a + 2] < coord[3 * b + 1] * NB2 + coord[3 * b + 2];
        });
        keys.resize(n);
        for (int i = 0; i < n; i++) keys[i] = (int)(coord[3 * tiles[i] + 1] * NB2 + coord[3 * tiles[i] + 2]);
        if (n) MPL_CUDA(cudaMemcpy(list.p, tiles.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
        return MPL_OK;
    };
    std::vector<int> lo_t, lo_k, hi_t, hi_k;
    MPL_CHECK(sorted(ctx->t_lo_list, ctx->n_lo_tiles, lo_t, lo_k));
    MPL_CHECK(sorted(ctx->t_hi_list, ctx->n_hi_tiles, hi_t, hi_k));
    const bool lo = ctx->rank > 0, hi = ctx->rank < ctx->nranks - 1;
    unsigned long long from_lo = 0, from_hi = 0;
    MPL_CHECK(exchange_counts(ctx, lo ? ctx->n_lo_tiles : 0, hi ? ctx->n_hi_tiles : 0, &from_lo, &from_hi));
    ctx->n_lo_recv = (int)from_lo;  // the lower neighbour's upper-face tiles
    ctx->n_hi_recv = (int)from_hi;  // the upper neighbour's lower-face tiles
    DevBuf ks_lo, ks_hi, kr_lo, kr_hi;
    auto cleanup = [&]() {
        for (DevBuf *b : {&ks_lo, &ks_hi, &kr_lo, &kr_hi})
            if (b->p) cudaFree(b->p);
    };
    std::vector<int> rl(ctx->n_lo_recv), rh(ctx->n_hi_recv);
    {
        mpl_status e = MPL_OK;
        if (ensure(ctx, ks_lo, lo_k.size() * 4 + 16) || ensure(ctx, ks_hi, hi_k.size() * 4 + 16) ||
            ensure(ctx, kr_lo, rl.size() * 4 + 16) || ensure(ctx, kr_hi, rh.size() * 4 + 16))
            e = MPL_ERR_OOM;
        if (e == MPL_OK && !lo_k.empty()) e = cudaMemcpy(ks_lo.p, lo_k.data(), lo_k.size() * 4, cudaMemcpyHostToDevice) ? MPL_ERR_CUDA : MPL_OK;
        if (e == MPL_OK && !hi_k.empty()) e = cudaMemcpy(ks_hi.p, hi_k.data(), hi_k.size() * 4, cudaMemcpyHostToDevice) ? MPL_ERR_CUDA : MPL_OK;
        if (e == MPL_OK)
            e = ctx->comm->neighbors(ctx, ks_lo.p, lo ? lo_k.size() * 4 : 0, kr_lo.p, lo ? rl.size() * 4 : 0, ks_hi.p,
                                     hi ? hi_k.size() * 4 : 0, kr_hi.p, hi ? rh.size() * 4 : 0);
        if (e == MPL_OK && !rl.empty()) e = cudaMemcpy(rl.data(), kr_lo.p, rl.size() * 4, cudaMemcpyDeviceToHost) ? MPL_ERR_CUDA : MPL_OK;
        if (e == MPL_OK && !rh.empty()) e = cudaMemcpy(rh.data(), kr_hi.p, rh.size() * 4, cudaMemcpyDeviceToHost) ? MPL_ERR_CUDA : MPL_OK;
        cleanup();
        if (e != MPL_OK) return e;
    }
    // received keys (sorted) -> local tile of the same (by, bz) on that face, or -1
    auto match = [&](const std::vector<int> &recv, const std::vector<int> &keys, const std::vector<int> &tiles,
                     DevBuf &map) -> mpl_status {
        std::vector<int> m(recv.size(), -1);
        size_t j = 0;
        for (size_t i = 0; i < recv.size(); i++) {
            while (j < keys.size() && keys[j] < recv[i]) j++;
            if (j < keys.size() && keys[j] == recv[i]) m[i] = tiles[j];
        }
        MPL_CHECK(ensure(ctx, map, m.size() * 4 + 16));
        if (!m.empty()) MPL_CUDA(cudaMemcpy(map.p, m.data(), m.size() * 4, cudaMemcpyHostToDevice));
        return MPL_OK;
    };
    MPL_CHECK(match(rl, lo_k, lo_t, ctx->t_lo_map));
    MPL_CHECK(match(rh, hi_k, hi_t, ctx->t_hi_map));
    // HVP split for the overlapped halo: the tiles at node-block x in {lo - 1, lo, hi - 1, hi} write the
    // shared planes (cells of the first / last owned block, the owned masses on the planes); no other tile
    // touches a shared-plane node
    {
        std::vector<int> bnd, inn;
        for (int t = 0; t < T_; t++) {
            const int bx = coord[3 * t];
            const bool b = bx == ctx->slab_lo - 1 || bx == ctx->slab_lo || bx == ctx->slab_hi - 1 || bx == ctx->slab_hi;
            (b ? bnd : inn).push_back(t);
        }
        ctx->n_bnd = (int)bnd.size();
        ctx->n_int = (int)inn.size();
        MPL_CHECK(ensure(ctx, ctx->t_bnd, bnd.size() * 4 + 16));
        MPL_CHECK(ensure(ctx, ctx->t_int, inn.size() * 4 + 16));
        if (!bnd.empty()) MPL_CUDA(cudaMemcpy(ctx->t_bnd.p, bnd.data(), bnd.size() * 4, cudaMemcpyHostToDevice));
        if (!inn.empty()) MPL_CUDA(cudaMemcpy(ctx->t_int.p, inn.data(), inn.size() * 4, cudaMemcpyHostToDevice));
    }
    return MPL_OK;
}

bool comm_is_nccl(mpl_ctx ctx) { return ctx->comm && dynamic_cast<NcclComm *>(ctx->comm) != nullptr; }

namespace {
// compact face buffers: send = this rank's face tiles, recv = the neighbour's (16 nodes x nv vectors each)
template <class T>
mpl_status ensure_faces(mpl_ctx ctx, int nv) {
    const size_t per = (size_t)16 * nv * sizeof(vec4<T>);
    MPL_CHECK(ensure(ctx, ctx->pl_send_lo, per * ctx->n_lo_tiles + 16));
    MPL_CHECK(ensure(ctx, ctx->pl_send_hi, per * ctx->n_hi_tiles + 16));
    MPL_CHECK(ensure(ctx, ctx->pl_recv_lo, per * ctx->n_lo_recv + 16));
    MPL_CHECK(ensure(ctx, ctx->pl_recv_hi, per * ctx->n_hi_recv + 16));
    return MPL_OK;
}
}  // namespace

// Sum of the partials of a (and b) on the shared node planes: pack this rank's face tiles (plane
// lx = 0 of the lower and upper face lists), exchange with both neighbours, add what arrives into the
// matching local tiles.  Bytes per message: 16 nodes x nv x 16 B (fp32) per face tile.
template <class T>
mpl_status halo_sum_nodes(mpl_ctx ctx, void *a_tile, void *b_tile) {
    if (!multi(ctx)) return MPL_OK;
    const int nv = b_tile ? 2 : 1;
    MPL_CHECK(ensure_faces<T>(ctx, nv));
    cudaStream_t st = ctx->stream;
    const size_t per = (size_t)16 * nv * sizeof(vec4<T>);
    const bool lo = ctx->rank > 0, hi = ctx->rank < ctx->nranks - 1;
    if (lo && ctx->n_lo_tiles)
        k_face_pack<T><<<ctx->n_lo_tiles, 16, 0, st>>>((const int *)ctx->t_lo_list.p, 0, nv, (const vec4<T> *)a_tile,
                                                       (const vec4<T> *)b_tile, (vec4<T> *)ctx->pl_send_lo.p),
            ctx->launches++;
    if (hi && ctx->n_hi_tiles)
        k_face_pack<T><<<ctx->n_hi_tiles, 16, 0, st>>>((const int *)ctx->t_hi_list.p, 0, nv, (const vec4<T> *)a_tile,
                                                       (const vec4<T> *)b_tile, (vec4<T> *)ctx->pl_send_hi.p),
            ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(ctx->comm->neighbors(ctx, ctx->pl_send_lo.p, lo ? per * ctx->n_lo_tiles : 0, ctx->pl_recv_lo.p,
                                   lo ? per * ctx->n_lo_recv : 0, ctx->pl_send_hi.p, hi ? per * ctx->n_hi_tiles : 0,
                                   ctx->pl_recv_hi.p, hi ? per * ctx->n_hi_recv : 0));
    if (lo && ctx->n_lo_recv)
        k_face_unpack<T, 0><<<ctx->n_lo_recv, 16, 0, st>>>((const int *)ctx->t_lo_map.p, 0, nv,
                                                           (const vec4<T> *)ctx->pl_recv_lo.p, (vec4<T> *)a_tile,
                                                           (vec4<T> *)b_tile),
            ctx->launches++;
    if (hi && ctx->n_hi_recv)
        k_face_unpack<T, 0><<<ctx->n_hi_recv, 16, 0, st>>>((const int *)ctx->t_hi_map.p, 0, nv,
                                                           (const vec4<T> *)ctx->pl_recv_hi.p, (vec4<T> *)a_tile,
                                                           (vec4<T> *)b_tile),
            ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

// G2P ghosts: the upper neighbour's second node plane (x = 4 X_{r+1} + 1, its lower face at lx = 1)
template <class T>
mpl_status ghost_nodes_from_upper(mpl_ctx ctx, void *v_tile) {
    if (!multi(ctx)) return MPL_OK;
    MPL_CHECK(ensure_faces<T>(ctx, 1));
    cudaStream_t st = ctx->stream;
    const size_t per = (size_t)16 * sizeof(vec4<T>);
    const bool lo = ctx->rank > 0, hi = ctx->rank < ctx->nranks - 1;
    if (lo && ctx->n_lo_tiles)
        k_face_pack<T><<<ctx->n_lo_tiles, 16, 0, st>>>((const int *)ctx->t_lo_list.p, 1, 1, (const vec4<T> *)v_tile,
                                                       nullptr, (vec4<T> *)ctx->pl_send_lo.p),
            ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(ctx->comm->neighbors(ctx, ctx->pl_send_lo.p, lo ? per * ctx->n_lo_tiles : 0, nullptr, 0, nullptr, 0,
                                   ctx->pl_recv_hi.p, hi ? per * ctx->n_hi_recv : 0));
    if (hi && ctx->n_hi_recv)
        k_face_unpack<T, 1><<<ctx->n_hi_recv, 16, 0, st>>>((const int *)ctx->t_hi_map.p, 1, 1,
                                                           (const vec4<T> *)ctx->pl_recv_hi.p, (vec4<T> *)v_tile,
                                                           nullptr),
            ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}

// (mv, m) partials in n_vn (w = m) -> completed on the shared planes; owner flags of the upper plane
template <class T>
mpl_status c2n_halo(mpl_ctx ctx) {
    if (!multi(ctx)) return MPL_OK;
    MPL_CHECK(ensure_faces<T>(ctx, 1));
    cudaStream_t st = ctx->stream;
    const size_t per = (size_t)16 * sizeof(vec4<T>);
    const bool lo = ctx->rank > 0, hi = ctx->rank < ctx->nranks - 1;
    vec4<T> *mvm = (vec4<T> *)ctx->n_vn.p;
    if (lo && ctx->n_lo_tiles)
        k_face_pack<T><<<ctx->n_lo_tiles, 16, 0, st>>>((const int *)ctx->t_lo_list.p, 0, 1, mvm, nullptr,
                                                       (vec4<T> *)ctx->pl_send_lo.p),
            ctx->launches++;
    if (hi && ctx->n_hi_tiles)
        k_face_pack<T><<<ctx->n_hi_tiles, 16, 0, st>>>((const int *)ctx->t_hi_list.p, 0, 1, mvm, nullptr,
                                                       (vec4<T> *)ctx->pl_send_hi.p),
            ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    MPL_CHECK(ctx->comm->neighbors(ctx, ctx->pl_send_lo.p, lo ? per * ctx->n_lo_tiles : 0, ctx->pl_recv_lo.p,
                                   lo ? per * ctx->n_lo_recv : 0, ctx->pl_send_hi.p, hi ? per * ctx->n_hi_tiles : 0,
                                   ctx->pl_recv_hi.p, hi ? per * ctx->n_hi_recv : 0));
    if (lo && ctx->n_lo_recv)
        k_c2n_face_unpack<T><<<ctx->n_lo_recv, 16, 0, st>>>((const int *)ctx->t_lo_map.p, 0,
                                                            (const vec4<T> *)ctx->pl_recv_lo.p, mvm,
                                                            (uint8_t *)ctx->n_own.p),
            ctx->launches++;
    if (hi && ctx->n_hi_recv)
        k_c2n_face_unpack<T><<<ctx->n_hi_recv, 16, 0, st>>>((const int *)ctx->t_hi_map.p, 1,
                                                            (const vec4<T> *)ctx->pl_recv_hi.p, mvm,
                                                            (uint8_t *)ctx->n_own.p),
            ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    return MPL_OK;
}


// Start of every resample on a slab rank: drop last step's ghosts, send particles that left the slab
// to the neighbour that now owns them, then copy the last owned cell plane to the upper neighbour as
// its ghosts.  Particle state moves to the other buffer set (cur flips).
template <class T>
mpl_status redistribute_particles(mpl_ctx ctx) {
    if (!multi(ctx)) {
        ctx->np_own = ctx->np;
        return MPL_OK;
    }
    cudaStream_t st = ctx->stream;
    const GridP &g = ctx->grid;
    const int64_t n = ctx->np;
    const int c = ctx->cur, nx = 1 - c;
    const int R = ctx->nranks, r = ctx->rank;
    const int A = 4 * ctx->cuts[r], B = 4 * ctx->cuts[r + 1];
    const int A_lo = r > 0 ? 4 * ctx->cuts[r - 1] : A, B_hi = r < R - 1 ? 4 * ctx->cuts[r + 2] : B;
    const size_t RB = rec_bytes<T>();
    MPL_CHECK(ensure(ctx, ctx->mig_cnt, 256));
    unsigned long long *cnt = (unsigned long long *)ctx->mig_cnt.p;  // [0..3] classes, [4..7] cursors
    int *bad = (int *)(cnt + 16);
    MPL_CUDA(cudaMemsetAsync(cnt, 0, 64, st));
    const int big = 0x7fffffff;
    MPL_CUDA(cudaMemcpyAsync(bad, &big, 4, cudaMemcpyHostToDevice, st));
    MPL_CHECK(ensure(ctx, ctx->pkey, (size_t)n * 4 + 16));
    if (n)
        k_classify<T><<<nblk(n, 256), 256, 0, st>>>(g, n, (const T *)ctx->px[c].p, (const int *)ctx->pid[c].p, A_lo, A, B,
                                                     B_hi, (int *)ctx->pkey.p, cnt, bad), ctx->launches++;
    unsigned long long h[4];
    int hbad = 0;
    MPL_CUDA(cudaMemcpyAsync(h, cnt, 32, cudaMemcpyDeviceToHost, st));
    MPL_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
    MPL_CUDA(cudaStreamSynchronize(st));
    // every rank takes part in the exchanges even when it fails, then reports
    unsigned long long in_lo = 0, in_hi = 0;
    DBG_GUARDS("redistribute: classify");
    MPL_CHECK(exchange_counts(ctx, h[1], h[2], &in_lo, &in_hi));
    MPL_CHECK(ensure(ctx, ctx->mig_send_lo, h[1] * RB + 16));
    MPL_CHECK(ensure(ctx, ctx->mig_send_hi, h[2] * RB + 16));
    MPL_CHECK(ensure(ctx, ctx->mig_recv_lo, in_lo * RB + 16));
    MPL_CHECK(ensure(ctx, ctx->mig_recv_hi, in_hi * RB + 16));
    const int64_t n_own = (int64_t)(h[0] + in_lo + in_hi);
    // destination buffers (content not needed): owned + room for ghosts
    const size_t s = sizeof(T);
    const int64_t cap = n_own + n_own / 4 + 1024;
    MPL_CHECK(ensure(ctx, ctx->px[nx], cap * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->pF[nx], cap * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->pv_alt, cap * 3 * s));
    MPL_CHECK(ensure(ctx, ctx->pG_alt, cap * 9 * s));
    MPL_CHECK(ensure(ctx, ctx->pvol[nx], cap * s));
    MPL_CHECK(ensure(ctx, ctx->pmat[nx], cap * 4));
    MPL_CHECK(ensure(ctx, ctx->pid[nx], cap * 4));
    PartOut o{ctx->px[nx].p, ctx->pv_alt.p, ctx->pF[nx].p, ctx->pG_alt.p, ctx->pvol[nx].p, (int *)ctx->pmat[nx].p,
              (int *)ctx->pid[nx].p};
    MPL_CUDA(cudaMemsetAsync(cnt + 4, 0, 32, st));
    if (n)
        k_migrate_pack<T><<<nblk(n, 256), 256, 0, st>>>(
            n, (const int *)ctx->pkey.p, (const T *)ctx->px[c].p, (const T *)ctx->pv.p, (const T *)ctx->pF[c].p,
            (const T *)ctx->pG.p, (const T *)ctx->pvol[c].p, (const int *)ctx->pmat[c].p, (const int *)ctx->pid[c].p,
            o, (char *)ctx->mig_send_lo.p, (char *)ctx->mig_send_hi.p, cnt + 4), ctx->launches++;
    MPL_CUDA(cudaGetLastError());
    DBG_GUARDS("redistribute: migrate pack");
    MPL_CHECK(ctx->comm->neighbors(ctx, ctx->mig_send_lo.p, h[1] * RB, ctx->mig_recv_lo.p, in_lo * RB,
                                   ctx->mig_send_hi.p, h[2] * RB, ctx->mig_recv_hi.p, in_hi * RB));
    if (in_lo)
        k_unpack_recs<T><<<nblk(in_lo, 256), 256, 0, st>>>((int64_t)in_lo, (const char *)ctx->mig_recv_lo.p,
                                                           (int64_t)h[0], 0, o), ctx->launches++;
    if (in_hi)
        k_unpack_recs<T><<<nblk(in_hi, 256), 256, 0, st>>>((int64_t)in_hi, (const char *)ctx->mig_recv_hi.p,
                                                           (int64_t)(h[0] + in_lo), 0, o), ctx->launches++;
    DBG_GUARDS("redistribute: migrant unpack");
    // ghosts: owned particles of cell plane B-1 go to the upper neighbour
    unsigned long long ng = 0;
    if (r < R - 1) {
        MPL_CUDA(cudaMemsetAsync(cnt + 8, 0, 8, st));
        if (n_own)
            k_count_plane<T><<<nblk(n_own, 256), 256, 0, st>>>(g, n_own, B - 1, (const T *)o.x, cnt + 8), ctx->launches++;
        MPL_CUDA(cudaMemcpyAsync(&ng, cnt + 8, 8, cudaMemcpyDeviceToHost, st));
        MPL_CUDA(cudaStreamSynchronize(st));
    }
    DBG_GUARDS("redistribute: ghost count");
    unsigned long long g_lo = 0, g_hi = 0;
    MPL_CHECK(exchange_counts(ctx, 0, ng, &g_lo, &g_hi));
    MPL_CHECK(ensure(ctx, ctx->mig_send_hi, ng * RB + 16));
    MPL_CHECK(ensure(ctx, ctx->mig_recv_lo, g_lo * RB + 16));
    if (ng) {
        MPL_CUDA(cudaMemsetAsync(cnt + 9, 0, 8, st));
        k_ghost_pack<T><<<nblk(n_own, 256), 256, 0, st>>>(g, n_own, B - 1, (const T *)o.x, (const T *)o.v,
                                                          (const T *)o.F, (const T *)o.G, (const T *)o.vol, o.mat, o.pid,
                                                          (char *)ctx->mig_send_hi.p, cnt + 9), ctx->launches++;
    }
    MPL_CUDA(cudaGetLastError());
    DBG_GUARDS("redistribute: ghost pack");
    MPL_CHECK(ctx->comm->neighbors(ctx, nullptr, 0, ctx->mig_recv_lo.p, g_lo * RB, ctx->mig_send_hi.p, ng * RB,
                                   nullptr, 0));
    const int64_t ntot = n_own + (int64_t)g_lo;
    if ((int64_t)cap < ntot) {
        // more ghosts than the headroom (a slab that starts nearly empty): grow the destination set,
        // keeping the n_own particles already unpacked into it
        const int64_t cap2 = ntot + ntot / 4 + 1024;
        MPL_CUDA(cudaStreamSynchronize(st));
        auto grow = [&](DevBuf &b, size_t per) -> mpl_status {
            DevBuf nb;
            MPL_CHECK(ensure(ctx, nb, (size_t)cap2 * per));
            if (n_own) MPL_CUDA(cudaMemcpy(nb.p, b.p, (size_t)n_own * per, cudaMemcpyDeviceToDevice));
            if (b.p) cudaFree(b.p);
            b = nb;
            return MPL_OK;
        };
        MPL_CHECK(grow(ctx->px[nx], 3 * s));
        MPL_CHECK(grow(ctx->pF[nx], 9 * s));
        MPL_CHECK(grow(ctx->pv_alt, 3 * s));
        MPL_CHECK(grow(ctx->pG_alt, 9 * s));
        MPL_CHECK(grow(ctx->pvol[nx], s));
        MPL_CHECK(grow(ctx->pmat[nx], 4));
        MPL_CHECK(grow(ctx->pid[nx], 4));
        o = PartOut{ctx->px[nx].p, ctx->pv_alt.p, ctx->pF[nx].p, ctx->pG_alt.p, ctx->pvol[nx].p, (int *)ctx->pmat[nx].p,
                    (int *)ctx->pid[nx].p};
    }
    if (g_lo)
        k_unpack_recs<T><<<nblk(g_lo, 256), 256, 0, st>>>((int64_t)g_lo, (const char *)ctx->mig_recv_lo.p, n_own, 1, o),
            ctx->launches++;
    DBG_GUARDS("redistribute: ghost unpack");
    MPL_CUDA(cudaGetLastError());
    MPL_CUDA(cudaStreamSynchronize(st));
    mpl_status bad_st = MPL_OK;
    if (hbad != big) {
        ctx->err = "particle " + std::to_string(hbad) + " left the slab by more than one neighbour (or the grid)";
        bad_st = MPL_ERR_OUT_OF_DOMAIN;
    }
    MPL_CHECK(agree(ctx, bad_st));
    std::swap(ctx->pv, ctx->pv_alt);
    std::swap(ctx->pG, ctx->pG_alt);
    ctx->cur = nx;
    ctx->np = ntot;
    ctx->np_own = n_own;
    return MPL_OK;
}

template <class T>
mpl_status export_owned_particles(mpl_ctx ctx, void *x, void *v, void *F, void *G, int32_t *ids, int32_t *base_ijk) {
    if (v || G) MPL_CHECK(sync_vg_order<T>(ctx));
    cudaStream_t st = ctx->stream;
    const int64_t n = ctx->np;
    const int c = ctx->cur;
    DevBuf keys, idx, keys2, idx2, tmp, out;
    auto cleanup = [&]() {
        for (DevBuf *b : {&keys, &idx, &keys2, &idx2, &tmp, &out})
            if (b->p) cudaFree(b->p);
    };
    size_t need = (size_t)n * 4 + 16;
    if (cudaMalloc(&keys.p, need) || cudaMalloc(&idx.p, need) || cudaMalloc(&keys2.p, need) ||
        cudaMalloc(&idx2.p, need) || cudaMalloc(&out.p, (size_t)n * 9 * sizeof(T) + 16)) {
        cudaGetLastError();
        cleanup();
        ctx->err = "out of device memory in particle export";
        return MPL_ERR_OOM;
    }
    MPL_CHECK(ensure(ctx, ctx->mig_cnt, 256));
    unsigned long long *cnt = (unsigned long long *)ctx->mig_cnt.p + 20;
    MPL_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
    if (n) k_owned_keys<<<nblk(n, 256), 256, 0, st>>>(n, (const int *)ctx->pid[c].p, (int *)keys.p, (int *)idx.p, cnt);
    unsigned long long m = 0;
    MPL_CUDA(cudaMemcpyAsync(&m, cnt, 8, cudaMemcpyDeviceToHost, st));
    MPL_CUDA(cudaStreamSynchronize(st));
    if ((int64_t)m != ctx->np_own) {
        cleanup();
        ctx->err = "particle export: " + std::to_string(m) + " owned particles found, expected " +
                   std::to_string(ctx->np_own) + " (np " + std::to_string(n) + ")";
        return MPL_ERR_STATE;
    }
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int *)keys.p, (int *)keys2.p, (const int *)idx.p, (int *)idx2.p,
                                    (int)m, 0, 32, st);
    if (cudaMalloc(&tmp.p, tb + 16)) {
        cudaGetLastError();
        cleanup();
        return MPL_ERR_OOM;
    }
    if (m)
        cub::DeviceRadixSort::SortPairs(tmp.p, tb, (const int *)keys.p, (int *)keys2.p, (const int *)idx.p,
                                        (int *)idx2.p, (int)m, 0, 32, st);
    struct Item { void *dst; const void *src; int w; };
    Item items[4] = {{x, ctx->px[c].p, 3}, {v, ctx->pv.p, 3}, {F, ctx->pF[c].p, 9}, {G, ctx->pG.p, 9}};
    for (auto &it : items) {
        if (!it.dst || !m) continue;
        k_gather_rows<T><<<nblk((int64_t)m * it.w, 256), 256, 0, st>>>((int64_t)m, it.w, (const int *)idx2.p,
                                                                        (const T *)it.src, (T *)out.p);
        cudaMemcpyAsync(it.dst, out.p, m * it.w * sizeof(T), cudaMemcpyDefault, st);
    }
    if (ids && m) cudaMemcpyAsync(ids, keys2.p, m * 4, cudaMemcpyDefault, st);
    if (base_ijk && m) {
        k_base_rows<<<nblk((int64_t)m, 256), 256, 0, st>>>((int64_t)m, (const int *)idx2.p, (const int *)ctx->pskey.p,
                                                          (const int *)ctx->t_coord.p, (int32_t *)out.p);
        cudaMemcpyAsync(base_ijk, out.p, m * 12, cudaMemcpyDefault, st);
    }
    cudaError_t e = cudaStreamSynchronize(st);
    cleanup();
    if (e != cudaSuccess) {
        ctx->err = std::string("CUDA error in particle export: ") + cudaGetErrorString(e);
        return MPL_ERR_CUDA;
    }
    return MPL_OK;
}

// =============================================================================================
// C ABI: groups, NCCL ids, slab cuts
// =============================================================================================
extern "C" {

mpl_status mpl_group_create(int32_t nranks, mpl_group *out) {
    if (!out || nranks < 1 || nranks > MAX_LOOPBACK) return MPL_ERR_INVALID_ARG;
    mpl_group g = new mpl_group_s();
    g->R = nranks;
    g->pa.assign(nranks, nullptr);
    g->pb.assign(nranks, nullptr);
    g->sa.assign(nranks, 0);
    g->sb.assign(nranks, 0);
    *out = g;
    return MPL_OK;
}

void mpl_group_destroy(mpl_group g) { delete g; }

mpl_status mpl_nccl_unique_id(uint8_t out[128]) {
    if (!out) return MPL_ERR_INVALID_ARG;
    NcclApi &api = nccl();
    if (!api.ok) return MPL_ERR_NCCL;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return MPL_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    memcpy(out, &id, 128);
    return MPL_OK;
}

// One-rank NCCL self-test on `device`: the exact entry points the slab transport uses (unique id,
// communicator init, in-place fp64 allreduce, a grouped send/receive to itself, destroy), so the
// dlopen'ed NCCL path is exercised on a single GPU (multi-rank runs need one GPU per rank).
mpl_status mpl_nccl_selftest(int32_t device, double *out_sum) {
    NcclApi &api = nccl();
    if (!api.ok) return MPL_ERR_NCCL;
    if (cudaSetDevice(device) != cudaSuccess) return MPL_ERR_CUDA;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return MPL_ERR_NCCL;
    ncclComm_t comm = nullptr;
    if (api.CommInitRank(&comm, 1, id, 0) != ncclSuccess) return MPL_ERR_NCCL;
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    double h[4] = {1.5, 2.5, 0.0, 0.0}, *d = nullptr;
    mpl_status rc = MPL_OK;
    if (cudaMalloc(&d, 4 * sizeof(double)) != cudaSuccess) rc = MPL_ERR_OOM;
    if (rc == MPL_OK) {
        cudaMemcpy(d, h, 4 * sizeof(double), cudaMemcpyHostToDevice);
        if (api.AllReduce(d, d, 2, ncclFloat64, ncclSum, comm, st) != ncclSuccess) rc = MPL_ERR_NCCL;
        if (rc == MPL_OK && (api.GroupStart() != ncclSuccess || api.Send(d, 16, ncclUint8, 0, comm, st) != ncclSuccess ||
                             api.Recv(d + 2, 16, ncclUint8, 0, comm, st) != ncclSuccess || api.GroupEnd() != ncclSuccess))
            rc = MPL_ERR_NCCL;
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = MPL_ERR_CUDA;
        cudaMemcpy(h, d, 4 * sizeof(double), cudaMemcpyDeviceToHost);
        cudaFree(d);
    }
    cudaStreamDestroy(st);
    api.CommDestroy(comm);
    if (out_sum) *out_sum = h[0] + h[1] + h[2] + h[3];  // 1.5 + 2.5 copied once more: 8.0
    return rc;
}

// Balanced slab cuts: cuts[0] = 0, cuts[nranks] = nplanes, and cuts[r] the first plane whose prefix
// weight reaches r/nranks of the total, kept strictly increasing (every slab >= 1 plane).
mpl_status mpl_balance_slabs(int32_t nplanes, const int64_t *weight, int32_t nranks, int32_t *cuts) {
    if (nplanes < 1 || nranks < 1 || nranks > nplanes || !cuts) return MPL_ERR_INVALID_ARG;
    std::vector<double> pre(nplanes + 1, 0.0);
    for (int p = 0; p < nplanes; p++) {
        const int64_t w = weight ? weight[p] : 1;
        if (w < 0) return MPL_ERR_INVALID_ARG;
        pre[p + 1] = pre[p] + (double)w;
    }
    const double tot = pre[nplanes];
    cuts[0] = 0;
    cuts[nranks] = nplanes;
    for (int r = 1; r < nranks; r++) {
        int c;
        if (tot <= 0) {
            c = (int)((int64_t)r * nplanes / nranks);
        } else {
            const double target = tot * r / nranks;
            c = 1;
            while (c < nplanes && pre[c] < target) c++;
            // nearer of c-1 and c
            if (c - 1 >= 1 && target - pre[c - 1] < pre[c] - target) c--;
        }
        const int lo = cuts[r - 1] + 1, hi = nplanes - (nranks - r);
        cuts[r] = c < lo ? lo : (c > hi ? hi : c);
    }
    return MPL_OK;
}

}  // extern "C"

template mpl_status redistribute_particles<float>(mpl_ctx);
template mpl_status redistribute_particles<double>(mpl_ctx);
template mpl_status halo_sum_nodes<float>(mpl_ctx, void *, void *);
template mpl_status halo_sum_nodes<double>(mpl_ctx, void *, void *);
template mpl_status ghost_nodes_from_upper<float>(mpl_ctx, void *);
template mpl_status ghost_nodes_from_upper<double>(mpl_ctx, void *);
template mpl_status c2n_halo<float>(mpl_ctx);
template mpl_status c2n_halo<double>(mpl_ctx);
template mpl_status export_owned_particles<float>(mpl_ctx, void *, void *, void *, void *, int32_t *, int32_t *);
template mpl_status export_owned_particles<double>(mpl_ctx, void *, void *, void *, void *, int32_t *, int32_t *);
