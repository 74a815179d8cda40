// libmht host runtime: plan loader, device layout, apply sequencing, C ABI.
//
// Loader (DESIGN.md §4 / §5):
//  1. stream the plan file once through two pinned 64 MiB buffers: factor
//     coefficients go straight to the device pool, the block tables and
//     index pools stay on the host; the u64 checksum is summed on the fly;
//  2. validate the chain invariant r_in(l,(t,v)) = r_out(l-1,(p,2v)) +
//     r_out(l-1,(p,2v+1)) and the leaf sizes;
//  3. resolve every block's input to <= 2 contiguous segments.  IDENTITY
//     blocks whose inputs are adjacent become aliases (no work, no bytes);
//     the others become COPY blocks.  This is where the level permutation is
//     fused into load addressing (north_star subsystem (2));
//  4. build size-sorted (LPT) forward row tiles and adjoint column tiles per
//     stage, and the adjoint group-sum pieces (sum-of-partials, no atomics);
//  5. upload the tables.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/mht.h"
#include "mht_internal.cuh"

using namespace mht;

namespace {
thread_local std::string g_err;

mht_status fail(mht_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? MHT_ERR_OOM : MHT_ERR_CUDA,           \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                       \
  } while (0)

struct FileBlock {
  int32_t kind, r_out, r_in, pad;
  int64_t idx_off, coef_off;
};
static_assert(sizeof(FileBlock) == 32, "block record");

struct Range {
  int32_t off = 0, count = 0;
};

}  // namespace

namespace mht {
// error reporting for the other translation units (mht_build.cu)
mht_status set_error(mht_status s, const char *msg) { return fail(s, msg); }
}  // namespace mht

struct mht_plan {
  int device = 0;
  cudaStream_t stream = nullptr;      // the stream applies are enqueued on
  cudaStream_t own_stream = nullptr;  // the plan's own (loader) stream, destroyed with the plan
  bool cplx = false;
  size_t ssz = 8;
  int64_t n = 0, m = 0;
  int L = 0;
  double tol = 0;
  int64_t plan_bytes = 0, factor_entries = 0, index_entries = 0, device_bytes = 0;
  int n_mat = 0, n_alias = 0;
  bool graphs = true;
  // CUDA-graph cache: one executable graph per (direction, nrhs, src, dst),
  // captured on an internal stream and launched on the caller's stream.
  struct GraphKey {
    int dir, nrhs;
    const void *src;
    void *dst;
    const double *diag;
    int diag_sqrt;
    bool operator<(const GraphKey &o) const {
      if (dir != o.dir) return dir < o.dir;
      if (nrhs != o.nrhs) return nrhs < o.nrhs;
      if (src != o.src) return src < o.src;
      if (dst != o.dst) return dst < o.dst;
      if (diag != o.diag) return diag < o.diag;
      return diag_sqrt < o.diag_sqrt;
    }
  };
  // coefficient-side diagonal of the current call (mht_apply_diag & co.)
  const double *cur_diag = nullptr;
  int cur_diag_sqrt = 0;
  void *d_ctmp = nullptr;  // m x nrhs scratch for mht_covariance_apply
  int ctmp_nrhs = 0;
  std::map<GraphKey, cudaGraphExec_t> gcache;
  cudaStream_t cap_stream = nullptr;
  void clear_graphs() {
    for (auto &kv : gcache) cudaGraphExecDestroy(kv.second);
    gcache.clear();
  }

  void *d_coef = nullptr;
  int32_t *d_idx = nullptr;
  int32_t *d_perm = nullptr;
  int32_t *d_permk = nullptr;  // plan v2 frequency permutation (nullptr: none)
  DevBlock *d_blocks = nullptr;
  Tile *d_fwd = nullptr;   // 64-row tiles (multi-RHS DMMA path)
  Tile *d_fwd1 = nullptr;  // nrhs = 1 tiles, with column splits on low-parallelism stages
  void *d_fsplit = nullptr;
  int *d_fcount = nullptr;
  Tile *d_adj = nullptr;
  Tile *d_adjm = nullptr;
  Piece *d_pieces = nullptr;
  int64_t *d_rd = nullptr;

  std::vector<Range> fwd, fwd1, adj, adjm, pieces;  // per stage 0..L+1
  // nrhs = 1 forward variant per stage: 1 = latency (fewer than two waves of
  // tiles at 7 CTAs per SM), 0 = streaming
  std::vector<char> fwd1_lat;
  std::vector<Range> pieces_u;  // pieces of the producers that are not fused (fused mode)
  // sharded plans (mht_plan_load_shard): G ranks, this is rank g, switch level ls;
  // exchange layout in zpool entries (x nrhs scalars each)
  int shard_G = 1, shard_g = 0, shard_ls = -1;
  std::vector<int64_t> send_off, send_len, recv_off, recv_len;
  // fused exchange (mht_shard_set_peers / mht_shard_open_peers): the zpool
  // allocation ends with a sync area ([2][G] arrival flags + 2 epochs) at
  // sync_byte_off; zrem / zdel as in Ctx, peer_sync[h] = rank h's sync area
  int64_t sync_byte_off = 0;
  bool x_on = false;
  int x_nrhs = 0;
  void **d_zrem = nullptr;
  int64_t *d_zdel = nullptr;
  unsigned long long **d_peersync = nullptr;
  std::vector<void *> ipc_open;  // peer mappings opened by mht_shard_open_peers
  int64_t *d_rdtab = nullptr;
  void *d_tmaps = nullptr;    // CUtensorMap per materialised block (complex adjoint TMA tiles)
  bool fused_sum = true;        // adjoint group sums on the consumer's load (MHT_FUSED_SUM=0: off)
  int n_unfused = 0;
  int64_t n_split_groups = 0;
  int64_t m_slabs = 0;    // multi-RHS adjoint split slabs (64 columns x nrhs each)
  int32_t m_groups = 0;   // multi-RHS adjoint split groups
  void *d_msplit = nullptr;
  int *d_mcount = nullptr;
  Range cpieces;
  std::vector<int64_t> stage_coef_bytes;
  std::vector<int32_t> stage_nmat;
  int64_t Zt = 0, Pt = 0;

  void *d_z = nullptr, *d_part = nullptr;
  int ws_nrhs = 0;
  void *d_hc = nullptr, *d_hf = nullptr;
  int host_nrhs = 0;
  // mht_apply_host_batch: copy streams (in / out), two device staging slots
  // (input and output buffers of max(m, n) x nrhs scalars each) and per-slot
  // events: input landed, transform done, output read back
  cudaStream_t s_in = nullptr, s_out = nullptr;
  void *d_bin[2] = {nullptr, nullptr}, *d_bout[2] = {nullptr, nullptr};
  int64_t bcap = 0;  // scalars per staging buffer
  cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
  // mht_lsqr work vectors (u, v, w, Phi v, Phi^* u, norm partials, per-column
  // state), kept across calls and grown with nrhs so repeated solves reuse the
  // same pointers (and the captured graphs keyed on them)
  void *lsqr_buf[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int lsqr_nrhs = 0;

  // profiling: one (start, stop) event pair per recorded launch
  struct Rec {
    int kind, stage, nrhs;
    cudaEvent_t a, b;
  };
  bool prof = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;

  ~mht_plan() {
    if (stream) cudaStreamSynchronize(stream);
    clear_graphs();
    if (own_stream && own_stream != stream) cudaStreamSynchronize(own_stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (void *q : ipc_open)
      if (q) cudaIpcCloseMemHandle(q);
    for (void *q : {(void *)d_zrem, (void *)d_zdel, (void *)d_peersync})
      if (q) cudaFree(q);
    for (cudaStream_t q : {s_in, s_out})
      if (q) {
        cudaStreamSynchronize(q);
        cudaStreamDestroy(q);
      }
    for (int i = 0; i < 2; ++i) {
      for (cudaEvent_t e : {ev_in[i], ev_comp[i], ev_out[i]})
        if (e) cudaEventDestroy(e);
      for (void *p : {d_bin[i], d_bout[i]})
        if (p) cudaFree(p);
    }
    if (own_stream) cudaStreamDestroy(own_stream);
    for (void *p : lsqr_buf)
      if (p) cudaFree(p);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (void *p : {(void *)d_coef, (void *)d_idx, (void *)d_perm, (void *)d_permk, (void *)d_blocks, (void *)d_fwd, (void *)d_fwd1, d_fsplit, (void *)d_fcount,
                    (void *)d_adj, (void *)d_adjm, (void *)d_pieces, (void *)d_rd, (void *)d_rdtab, d_msplit, (void *)d_mcount, d_ctmp, d_tmaps, d_z, d_part, d_hc, d_hf})
      if (p) cudaFree(p);
  }
};

namespace {

// ---------------------------------------------------------------- file IO
struct Reader {
  FILE *fp = nullptr;
  uint64_t csum = 0;
  int64_t body_read = 0;
  ~Reader() {
    if (fp) fclose(fp);
  }
  bool read(void *dst, size_t bytes, bool in_body = true) {
    if (bytes == 0) return true;
    if (fread(dst, 1, bytes, fp) != bytes) return false;
    if (in_body) {
      const uint64_t *w = static_cast<const uint64_t *>(dst);
      uint64_t s = 0;
      for (size_t i = 0; i < bytes / 8; ++i) s += w[i];
      csum += s;
      body_read += (int64_t)bytes;
    }
    return true;
  }
};

size_t pad8(size_t b) { return (b + 7) / 8 * 8; }

template <class T>
mht_status upload(T **dptr, const std::vector<T> &v, int64_t &acct) {
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  CUDA_TRY(cudaMalloc((void **)dptr, bytes));
  acct += (int64_t)bytes;
  if (!v.empty()) CUDA_TRY(cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return MHT_OK;
}

struct Loc {
  int32_t src = SRC_C;
  int64_t off = 0;
};

// Plan sharding: G ranks; stages 0..ls are partitioned by
// the G frequency subtrees at height L - log2 G, stages ls+1..L+1 by the G
// space subtrees at depth log2 G; one all-to-all of z_ls between the phases.
struct ShardCfg {
  int G = 1, g = 0, ls = -1;
};

mht_status load_impl(const char *path, int device, std::unique_ptr<mht_plan> &P, const ShardCfg &sh) {
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MHT_ERR_INVALID_ARG, "bad device ordinal");
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(MHT_ERR_UNSUPPORTED, "libmht is built for sm_100a (B200)");
  CUDA_TRY(cudaSetDevice(device));
  P->device = device;

  Reader R;
  R.fp = fopen(path, "rb");
  if (!R.fp) return fail(MHT_ERR_IO, std::string("cannot open ") + path);
  fseeko(R.fp, 0, SEEK_END);
  const int64_t fbytes = ftello(R.fp);
  fseeko(R.fp, 0, SEEK_SET);
  unsigned char hdr[256];
  if (fbytes < 256 || !R.read(hdr, 256, false)) return fail(MHT_ERR_FORMAT, "short header");
  if (memcmp(hdr, "BFMHTPLN", 8) != 0) return fail(MHT_ERR_FORMAT, "bad magic");
  uint32_t ver, dt;
  int64_t nst, body;
  uint64_t csum;
  int32_t L;
  memcpy(&ver, hdr + 8, 4);
  memcpy(&dt, hdr + 12, 4);
  memcpy(&P->n, hdr + 16, 8);
  memcpy(&P->m, hdr + 24, 8);
  memcpy(&L, hdr + 32, 4);
  memcpy(&P->tol, hdr + 40, 8);
  memcpy(&nst, hdr + 48, 8);
  memcpy(&csum, hdr + 56, 8);
  memcpy(&body, hdr + 64, 8);
  if (ver != 1 && ver != 2) return fail(MHT_ERR_FORMAT, "unsupported plan version");
  if (dt != 1 && dt != 2) return fail(MHT_ERR_FORMAT, "bad dtype");
  if (L < 0 || L > 24 || nst != L + 2) return fail(MHT_ERR_FORMAT, "bad L / stage count");
  if (body < 0 || body + 256 != fbytes) return fail(MHT_ERR_FORMAT, "body size mismatch");
  if (P->n < 1 || P->m < 1 || P->n > INT32_MAX || P->m > INT32_MAX) return fail(MHT_ERR_SHAPE, "bad n/m");
  P->L = L;
  P->cplx = dt == 2;
  P->ssz = P->cplx ? 16 : 8;
  P->plan_bytes = fbytes;
  const int64_t nl = int64_t(1) << L;

  std::vector<int32_t> perm((size_t)pad8(4 * P->n) / 4);
  std::vector<int64_t> sp_off(nl + 1), fr_off(nl + 1);
  if (!R.read(perm.data(), pad8(4 * P->n)) || !R.read(sp_off.data(), 8 * (nl + 1)) ||
      !R.read(fr_off.data(), 8 * (nl + 1)))
    return fail(MHT_ERR_FORMAT, "truncated trees");
  perm.resize(P->n);
  // version 2: the frequency permutation perm_k (plan position -> user c index)
  std::vector<int32_t> perm_k;
  if (ver == 2) {
    perm_k.resize(pad8(4 * P->m) / 4);
    if (!R.read(perm_k.data(), pad8(4 * P->m))) return fail(MHT_ERR_FORMAT, "truncated perm_k");
    perm_k.resize(P->m);
    std::vector<char> seen(P->m, 0);
    for (int32_t j : perm_k) {
      if (j < 0 || j >= P->m || seen[j]) return fail(MHT_ERR_FORMAT, "perm_k is not a permutation");
      seen[j] = 1;
    }
  }
  if (sp_off[0] != 0 || sp_off[nl] != P->n || fr_off[0] != 0 || fr_off[nl] != P->m)
    return fail(MHT_ERR_FORMAT, "tree offsets do not cover n / m");
  for (int64_t i = 0; i < nl; ++i)
    if (sp_off[i + 1] < sp_off[i] || fr_off[i + 1] < fr_off[i])
      return fail(MHT_ERR_FORMAT, "tree offsets not monotone");
  {
    std::vector<char> seen(P->n, 0);
    for (int32_t j : perm) {
      if (j < 0 || j >= P->n || seen[j]) return fail(MHT_ERR_FORMAT, "perm_x is not a permutation");
      seen[j] = 1;
    }
  }

  // device coefficient pool: the body size bounds the coefficient bytes.  A
  // shard reads only its own blocks' coefficients (second pass below).
  const bool sharded = sh.G > 1;
  CUDA_TRY(cudaStreamCreateWithFlags(&P->own_stream, cudaStreamNonBlocking));
  P->stream = P->own_stream;
  size_t pool_bytes = std::max<int64_t>(16, body);
  if (!sharded) {
    CUDA_TRY(cudaMalloc(&P->d_coef, pool_bytes));
    P->device_bytes += (int64_t)pool_bytes;
  }
  std::vector<int64_t> coef_file_off(L + 2, 0);  // file offset of each stage's coefficients

  const size_t CH = size_t(64) << 20;
  void *pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2];
  CUDA_TRY(cudaHostAlloc(&pin[0], CH, cudaHostAllocDefault));
  CUDA_TRY(cudaHostAlloc(&pin[1], CH, cudaHostAllocDefault));
  CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct PinGuard {
    void **p;
    cudaEvent_t *e;
    ~PinGuard() {
      cudaFreeHost(p[0]);
      cudaFreeHost(p[1]);
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } pg{pin, ev};
  int which = 0;
  bool pending[2] = {false, false};

  std::vector<std::vector<FileBlock>> blk(L + 2);
  std::vector<std::vector<int32_t>> idx(L + 2);
  std::vector<int64_t> coef_base(L + 2), ncoef_s(L + 2);
  int64_t coef_cursor = 0;  // in scalars
  for (int s = 0; s < L + 2; ++s) {
    int64_t sh[4];
    if (!R.read(sh, 32)) return fail(MHT_ERR_FORMAT, "truncated stage header");
    if (sh[0] != s || sh[1] != nl || sh[2] < 0 || sh[3] < 0) return fail(MHT_ERR_FORMAT, "bad stage header");
    const int64_t nidx = sh[2], ncoef = sh[3];
    if ((coef_cursor + ncoef) * (int64_t)P->ssz > (int64_t)pool_bytes) return fail(MHT_ERR_FORMAT, "coefficients overflow body");
    coef_base[s] = coef_cursor;
    ncoef_s[s] = ncoef;
    coef_file_off[s] = ftello(R.fp);
    int64_t left = ncoef * (int64_t)P->ssz;
    if (sharded && left > 0) {  // skip now; the shard's blocks are read after resolution
      if (fseeko(R.fp, left, SEEK_CUR) != 0 || ftello(R.fp) > fbytes) return fail(MHT_ERR_FORMAT, "truncated coefficients");
      R.body_read += left;
      left = 0;
    }
    char *dst = static_cast<char *>(P->d_coef) + coef_cursor * (int64_t)P->ssz;
    while (left > 0) {
      size_t b = (size_t)std::min<int64_t>(left, (int64_t)CH);
      if (pending[which]) CUDA_TRY(cudaEventSynchronize(ev[which]));
      if (!R.read(pin[which], b)) return fail(MHT_ERR_FORMAT, "truncated coefficients");
      CUDA_TRY(cudaMemcpyAsync(dst, pin[which], b, cudaMemcpyHostToDevice, P->stream));
      CUDA_TRY(cudaEventRecord(ev[which], P->stream));
      pending[which] = true;
      which ^= 1;
      dst += b;
      left -= (int64_t)b;
    }
    coef_cursor += ncoef;
    blk[s].resize(nl);
    if (!R.read(blk[s].data(), 32 * nl)) return fail(MHT_ERR_FORMAT, "truncated block table");
    idx[s].resize(pad8(4 * nidx) / 4);
    if (!R.read(idx[s].data(), pad8(4 * nidx))) return fail(MHT_ERR_FORMAT, "truncated index pool");
    idx[s].resize(nidx);
  }
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  if (R.body_read != body) return fail(MHT_ERR_FORMAT, "trailing bytes after last stage");
  // a shard does not read every coefficient, so it cannot verify the whole-body checksum
  if (!sharded && R.csum != csum) return fail(MHT_ERR_FORMAT, "checksum mismatch");
  P->factor_entries = coef_cursor;

  // ------------------------------------------------ validation
  auto bad_block = [&](int s, int64_t b, const char *why) {
    char buf[160];
    snprintf(buf, sizeof buf, "stage %d block %lld: %s", s, (long long)b, why);
    return fail(MHT_ERR_FORMAT, buf);
  };
  for (int s = 0; s < L + 2; ++s) {
    for (int64_t b = 0; b < nl; ++b) {
      const FileBlock &B = blk[s][b];
      if (B.r_out < 0 || B.r_in < 0) return bad_block(s, b, "negative size");
      int64_t want_in;
      if (s == 0) {
        want_in = fr_off[b + 1] - fr_off[b];
      } else if (s <= L) {
        const int64_t nf = nl >> s, nfp = nl >> (s - 1), t = b / nf, v = b % nf, p = t >> 1;
        want_in = (int64_t)blk[s - 1][p * nfp + 2 * v].r_out + blk[s - 1][p * nfp + 2 * v + 1].r_out;
      } else {
        want_in = blk[L][b].r_out;
        if (B.r_out != sp_off[b + 1] - sp_off[b]) return bad_block(s, b, "leaf rows != |tau|");
      }
      if (B.r_in != want_in) return bad_block(s, b, "chain invariant r_in = r(p,c1)+r(p,c2) violated");
      if (B.kind == 0) {
        if (B.r_out != B.r_in) return bad_block(s, b, "IDENTITY with r_out != r_in");
      } else if (B.kind == 1) {
        if (B.r_out > B.r_in) return bad_block(s, b, "ID with r_out > r_in");
        if (B.idx_off < 0 || B.idx_off + B.r_in > (int64_t)idx[s].size()) return bad_block(s, b, "index range");
        if (B.coef_off < 0 || B.coef_off + (int64_t)B.r_out * (B.r_in - B.r_out) > ncoef_s[s])
          return bad_block(s, b, "coefficient range");
        for (int i = 0; i < B.r_in; ++i) {
          int32_t q = idx[s][B.idx_off + i];
          if (q < 0 || q >= B.r_in) return bad_block(s, b, "index out of range");
        }
      } else if (B.kind == 2) {
        if (B.coef_off < 0 || B.coef_off + (int64_t)B.r_out * B.r_in > ncoef_s[s])
          return bad_block(s, b, "coefficient range");
      } else {
        return bad_block(s, b, "unknown kind");
      }
    }
  }

  // ------------------------------------------------ resolution
  std::vector<int32_t> idx_all;
  std::vector<int64_t> idx_base(L + 2);
  for (int s = 0; s < L + 2; ++s) {
    idx_base[s] = (int64_t)idx_all.size();
    idx_all.insert(idx_all.end(), idx[s].begin(), idx[s].end());
  }
  P->index_entries = (int64_t)idx_all.size();

  std::vector<DevBlock> blocks;
  std::vector<int> block_stage;
  struct RecvRegion {
    int64_t off, len;
    int32_t src;  // the sending rank
  };
  std::vector<RecvRegion> recv_regions;  // sharded: the exchange's receive buffer
  int64_t send_base = 0;
  std::vector<std::vector<Loc>> loc(L + 1, std::vector<Loc>(nl));
  int64_t Z = 0, Pp = 0;
  P->stage_coef_bytes.assign(L + 2, 0);
  P->stage_nmat.assign(L + 2, 0);
  auto materialize = [&](int s, const FileBlock &F, Loc a, int32_t la, Loc bb, int32_t lb, bool leaf,
                         int64_t leaf_row0) {
    DevBlock D;
    memset(&D, 0, sizeof D);
    D.seg_src[0] = a.src;
    D.seg_off[0] = a.off;
    D.seg_len[0] = la;
    D.seg_src[1] = bb.src;
    D.seg_off[1] = bb.off;
    D.seg_len[1] = lb;
    D.r_out = F.r_out;
    D.r_in = F.r_in;
    if (F.kind == 1) {
      D.n_skel = F.r_out;
      D.n_red = F.r_in - F.r_out;
      D.skel_off = idx_base[s] + F.idx_off;
      D.red_off = D.skel_off + F.r_out;
      D.coef_off = coef_base[s] + F.coef_off;
      P->stage_coef_bytes[s] += (int64_t)F.r_out * (F.r_in - F.r_out) * (int64_t)P->ssz;
    } else if (F.kind == 2) {
      D.n_skel = 0;
      D.n_red = F.r_in;
      D.flags |= F_RED_IOTA;
      D.coef_off = coef_base[s] + F.coef_off;
      P->stage_coef_bytes[s] += (int64_t)F.r_out * F.r_in * (int64_t)P->ssz;
    } else {  // COPY
      D.n_skel = F.r_in;
      D.n_red = 0;
      D.flags |= F_SKEL_IOTA;
    }
    if (leaf) {
      D.flags |= F_OUT_F;
      D.out_off = leaf_row0;
    } else {
      D.out_off = Z;
      Z += F.r_out;
    }
    D.part_off = Pp;
    Pp += F.r_in;
    blocks.push_back(D);
    block_stage.push_back(s);
    P->stage_nmat[s] += 1;
    return Loc{SRC_Z, D.out_off};
  };
  // ownership (sharded plans): stage s <= ls by frequency node v (height s),
  // stage s > ls by space node t (depth s); aligned subtrees, so a block's
  // inputs are local except the stage-(ls+1) reads of z_ls (the exchange)
  auto own_v = [&](int s, int64_t v) { return !sharded || v / ((nl >> s) / sh.G) == sh.g; };
  auto own_t = [&](int s, int64_t t) { return !sharded || t / ((int64_t(1) << s) / sh.G) == sh.g; };
  for (int64_t v = 0; v < nl; ++v) {
    if (!own_v(0, v)) continue;
    const FileBlock &F = blk[0][v];
    Loc c0{SRC_C, fr_off[v]};
    if (F.kind == 0 && !(sharded && sh.ls == 0)) {
      loc[0][v] = c0;
      P->n_alias++;
    } else {
      loc[0][v] = materialize(0, F, c0, F.r_in, Loc{SRC_C, 0}, 0, false, 0);
    }
  }
  if (sharded) {
    P->send_off.assign(sh.G, 0);
    P->send_len.assign(sh.G, 0);
    P->recv_off.assign(sh.G, 0);
    P->recv_len.assign(sh.G, 0);
  }
  for (int s = 1; s <= L; ++s) {
    const int64_t nf = nl >> s, nfp = nl >> (s - 1);
    const bool freq_phase = !sharded || s <= sh.ls;
    if (sharded && s == sh.ls) send_base = Z;
    for (int64_t b = 0; b < nl; ++b) {
      const int64_t t = b / nf, v = b % nf, p = t >> 1;
      if (freq_phase ? !own_v(s, v) : !own_t(s, t)) continue;
      const int64_t b1 = p * nfp + 2 * v, b2 = b1 + 1;
      const Loc A = loc[s - 1][b1], B = loc[s - 1][b2];
      const int32_t la = blk[s - 1][b1].r_out, lb = blk[s - 1][b2].r_out;
      const FileBlock &F = blk[s][b];
      // the switch stage's outputs are the send buffer: always materialised,
      // laid out destination by destination (t-major order)
      const bool send = sharded && s == sh.ls;
      int dest = -1;
      if (send) {
        const int h = (int)(t / ((int64_t(1) << s) / sh.G));
        dest = h;
        if (P->send_len[h] == 0) P->send_off[h] = Z;
        P->send_len[h] += F.r_out;
      }
      if (F.kind == 0 && !send) {
        if (lb == 0) {
          loc[s][b] = A;
          P->n_alias++;
          continue;
        }
        if (la == 0) {
          loc[s][b] = B;
          P->n_alias++;
          continue;
        }
        if (A.src == B.src && A.off + la == B.off) {
          loc[s][b] = A;
          P->n_alias++;
          continue;
        }
      }
      loc[s][b] = materialize(s, F, A, la, B, lb, false, 0);
      if (send) blocks.back().flags |= F_REMOTE | (dest << 16);
    }
    if (sharded && s == sh.ls) {
      // send regions are contiguous in destination order (t-major); give empty
      // destinations their position in the sequence
      int64_t run = send_base;
      for (int h = 0; h < sh.G; ++h) {
        P->send_off[h] = run;
        run += P->send_len[h];
      }
      if (run != Z) return fail(MHT_ERR_FORMAT, "shard send layout");
      // receive buffer: z_ls(t, v) for my space nodes t and every v, source by
      // source in the senders' order; the next stage reads it in place
      for (int src = 0; src < sh.G; ++src) {
        P->recv_off[src] = Z;
        for (int64_t t = 0; t < (int64_t(1) << s); ++t) {
          if (!own_t(s, t)) continue;
          for (int64_t v = 0; v < nf; ++v) {
            if (v / (nf / sh.G) != src) continue;
            loc[s][t * nf + v] = Loc{SRC_Z, Z};
            recv_regions.push_back({Z, (int64_t)blk[s][t * nf + v].r_out, (int32_t)src});
            Z += blk[s][t * nf + v].r_out;
          }
        }
        P->recv_len[src] = Z - P->recv_off[src];
      }
    }
  }
  for (int64_t t = 0; t < nl; ++t) {
    if (!own_t(L, t)) continue;
    const FileBlock &F = blk[L + 1][t];
    materialize(L + 1, F, loc[L][t], blk[L][t].r_out, Loc{SRC_C, 0}, 0, true, sp_off[t]);
  }
  P->Zt = std::max<int64_t>(Z, 1);
  P->Pt = std::max<int64_t>(Pp, 1);
  P->n_mat = (int)blocks.size();

  // ------------------------------------------------ shard: read this rank's coefficients
  if (sharded) {
    P->shard_G = sh.G;
    P->shard_g = sh.g;
    P->shard_ls = sh.ls;
    struct Job {
      int64_t file_off, nbytes;
      int blk;
    };
    std::vector<Job> jobs;
    int64_t total = 0;
    for (int i = 0; i < (int)blocks.size(); ++i) {
      DevBlock &D = blocks[i];
      if (D.n_red == 0 || D.r_out == 0) continue;
      const int st_ = block_stage[i];
      const int64_t within = D.coef_off - coef_base[st_];  // scalars into the stage's coefficients
      jobs.push_back({coef_file_off[st_] + within * (int64_t)P->ssz, (int64_t)D.r_out * D.n_red * (int64_t)P->ssz, i});
      total += jobs.back().nbytes;
    }
    std::sort(jobs.begin(), jobs.end(), [](const Job &a, const Job &b) { return a.file_off < b.file_off; });
    pool_bytes = (size_t)std::max<int64_t>(16, total);
    CUDA_TRY(cudaMalloc(&P->d_coef, pool_bytes));
    P->device_bytes += (int64_t)pool_bytes;
    int64_t cur = 0;  // device byte cursor
    for (const Job &j : jobs) {
      blocks[j.blk].coef_off = cur / (int64_t)P->ssz;
      if (fseeko(R.fp, j.file_off, SEEK_SET) != 0) return fail(MHT_ERR_IO, "seek");
      int64_t left = j.nbytes;
      char *dst = static_cast<char *>(P->d_coef) + cur;
      while (left > 0) {
        const size_t b = (size_t)std::min<int64_t>(left, (int64_t)CH);
        if (pending[which]) CUDA_TRY(cudaEventSynchronize(ev[which]));
        if (fread(pin[which], 1, b, R.fp) != b) return fail(MHT_ERR_FORMAT, "truncated coefficients");
        CUDA_TRY(cudaMemcpyAsync(dst, pin[which], b, cudaMemcpyHostToDevice, P->stream));
        CUDA_TRY(cudaEventRecord(ev[which], P->stream));
        pending[which] = true;
        which ^= 1;
        dst += b;
        left -= (int64_t)b;
      }
      cur += j.nbytes;
    }
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    P->factor_entries = total / (int64_t)P->ssz;
    coef_cursor = P->factor_entries;
  }

  // ------------------------------------------------ factor layout
  // Complex factors keep the file layout (16-byte scalars are always aligned).
  // Real factors are repacked on the device so every column of every block
  // starts 16-byte aligned (ld rounded up to even, zero pad row): the nrhs = 1
  // kernels then stream two rows per 16-byte load.
  for (DevBlock &D : blocks) D.ld = D.r_out;
  if (!P->cplx && coef_cursor > 0) {
    std::vector<Repack> jobs;
    int64_t cur = 0;
    for (DevBlock &D : blocks) {
      if (D.n_red == 0 || D.r_out == 0) continue;  // COPY / empty: no coefficients
      Repack J;
      memset(&J, 0, sizeof J);
      J.src_off = D.coef_off;
      J.dst_off = cur;
      J.r_out = D.r_out;
      J.ncols = D.n_red;
      J.dst_ld = D.r_out + (D.r_out & 1);
      D.coef_off = cur;
      D.ld = J.dst_ld;
      cur += (int64_t)J.dst_ld * J.ncols;
      cur += cur & 1;
      jobs.push_back(J);
    }
    void *np = nullptr;
    const size_t nbytes = (size_t)std::max<int64_t>(cur + 2, 16) * sizeof(double);  // +2: pair loads past the end
    CUDA_TRY(cudaMalloc(&np, nbytes));
    CUDA_TRY(cudaMemsetAsync(np, 0, nbytes, P->stream));
    Repack *dj = nullptr;
    CUDA_TRY(cudaMalloc((void **)&dj, std::max<size_t>(1, jobs.size()) * sizeof(Repack)));
    if (!jobs.empty()) {
      CUDA_TRY(cudaMemcpy(dj, jobs.data(), jobs.size() * sizeof(Repack), cudaMemcpyHostToDevice));
      launch_repack(static_cast<const double *>(P->d_coef), static_cast<double *>(np), dj, (int)jobs.size(), P->stream);
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    cudaFree(dj);
    cudaFree(P->d_coef);
    P->device_bytes -= (int64_t)pool_bytes;
    P->d_coef = np;
    P->device_bytes += (int64_t)nbytes;
  }

  // ------------------------------------------------ TMA descriptors (complex adjoint tiles)
  // One 2-D tensor map per block with coefficients: T viewed as a column-major
  // (2 r_out doubles) x n_red array of float64, row stride ld; box = 8 complex
  // rows (128 bytes) x 64 columns, 128-byte swizzle (half of the adjoint
  // tile's K chunk per request), out-of-range rows / columns zero-filled by
  // the TMA unit.  Real plans use no tensor maps.
  if (P->cplx) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void *fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (!encode) return fail(MHT_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    std::vector<CUtensorMap> maps(blocks.size());
    const int bk = P->cplx ? 16 : 32;
    const int ew = P->cplx ? 2 : 1;  // doubles per scalar
    for (size_t i = 0; i < blocks.size(); ++i) {
      const DevBlock &D = blocks[i];
      memset(&maps[i], 0, sizeof(CUtensorMap));
      if (D.n_red == 0 || D.r_out == 0) continue;
      cuuint64_t dims[2] = {(cuuint64_t)D.r_out * ew, (cuuint64_t)D.n_red};
      cuuint64_t strides[1] = {(cuuint64_t)D.ld * P->ssz};
      cuuint32_t box[2] = {(cuuint32_t)(bk * ew / 2), (cuuint32_t)MMA_COLS};  // 128-byte rows
      cuuint32_t estr[2] = {1, 1};
      void *addr = static_cast<char *>(P->d_coef) + D.coef_off * (int64_t)P->ssz;
      CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, addr, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        char buf[128];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) for block %zu", (int)r, i);
        return fail(MHT_ERR_CUDA, buf);
      }
    }
    CUDA_TRY(cudaMalloc(&P->d_tmaps, std::max<size_t>(1, maps.size()) * sizeof(CUtensorMap)));
    if (!maps.empty())
      CUDA_TRY(cudaMemcpy(P->d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    P->device_bytes += (int64_t)maps.size() * (int64_t)sizeof(CUtensorMap);
  }

  // ------------------------------------------------ tiles (LPT order per stage)
  std::vector<std::vector<std::pair<int64_t, Tile>>> ft(L + 2), at(L + 2), amt(L + 2);
  for (int i = 0; i < (int)blocks.size(); ++i) {
    const DevBlock &D = blocks[i];
    const int s = block_stage[i];
    for (int r0 = 0; r0 < D.r_out; r0 += FWD_ROWS) {
      int cnt = std::min(FWD_ROWS, D.r_out - r0);
      ft[s].push_back({(int64_t)cnt * (D.n_red + 4), Tile{i, r0, cnt, -1}});
    }
    if (D.n_red == 0) {
      amt[s].push_back({(int64_t)D.r_out + D.n_skel, Tile{i, 0, 0, -1}});
    } else {
      for (int c0 = 0; c0 < D.n_red; c0 += MMA_COLS) {
        int cnt = std::min(MMA_COLS, D.n_red - c0);
        const int ntl = (D.n_red + MMA_COLS - 1) / MMA_COLS;  // the skeleton copy is spread over the tiles
        amt[s].push_back({(int64_t)cnt * (D.r_out + 4) + (D.n_skel + ntl - 1) / ntl, Tile{i, c0, cnt, -1}});
      }
    }
    if (D.n_red == 0) {
      at[s].push_back({(int64_t)D.r_out + D.n_skel, Tile{i, 0, 0, -1}});
    } else {
      const int acols = P->cplx ? ADJ_COLS : ADJ_COLS_REAL;
      for (int c0 = 0; c0 < D.n_red; c0 += acols) {
        int cnt = std::min(acols, D.n_red - c0);
        at[s].push_back({(int64_t)cnt * (D.r_out + 4) + (c0 == 0 ? D.n_skel : 0), Tile{i, c0, cnt, -1}});
      }
    }
  }
  std::vector<Tile> fwd_all, adj_all, adjm_all;
  const int ADJ1_TARGET = prop.multiProcessorCount * 6;
  const int ADJ1_MIN_SPLIT = 128;
  int64_t asplit_scalars = 0;
  int32_t agroups = 0;
  const int MMA_TARGET = prop.multiProcessorCount * 4;
  const int MMA_MIN_SPLIT = 256;
  int64_t mslabs = 0;
  int32_t mgroups = 0;
  P->fwd.assign(L + 2, Range{});
  P->adj.assign(L + 2, Range{});
  P->adjm.assign(L + 2, Range{});
  auto by_cost = [](const std::pair<int64_t, Tile> &a, const std::pair<int64_t, Tile> &b) {
    return a.first > b.first;
  };
  for (int s = 0; s < L + 2; ++s) {
    std::stable_sort(ft[s].begin(), ft[s].end(), by_cost);
    P->fwd[s] = Range{(int32_t)fwd_all.size(), (int32_t)ft[s].size()};
    for (auto &x : ft[s]) fwd_all.push_back(x.second);
    // nrhs = 1 adjoint row splits: a stage with fewer column tiles than
    // ADJ1_TARGET splits the rows of its tall blocks (>= ADJ1_MIN_SPLIT rows
    // per split); partial column sums are combined by the group's last CTA.
    {
      const int nt = (int)at[s].size();
      std::vector<std::pair<int64_t, Tile>> lst;
      for (auto &x : at[s]) {
        DevBlock &D = blocks[x.second.blk];
        int ks = 1;
        if (nt > 0 && nt < ADJ1_TARGET && D.n_red > 0 && D.r_out >= 2 * ADJ1_MIN_SPLIT) {
          ks = (ADJ1_TARGET + nt - 1) / nt;
          ks = std::min(ks, D.r_out / ADJ1_MIN_SPLIT);
          ks = std::min(ks, 255);
        }
        if (ks <= 1 || x.second.count == 0) {
          lst.push_back(x);
          continue;
        }
        if (D.pad2 == 0) {  // first column tile of the block: reserve its scratch
          D.pad2 = ks;
          D.asp_off = asplit_scalars;
          const int acols = P->cplx ? ADJ_COLS : ADJ_COLS_REAL;
          asplit_scalars += (int64_t)((D.n_red + acols - 1) / acols) * ks * acols;
        }
        const int chunk = ((D.r_out + ks - 1) / ks + 31) & ~31;
        for (int k = 0; k < ks; ++k) {
          const int rows = std::max(0, std::min(D.r_out, (k + 1) * chunk) - k * chunk);
          Tile t = x.second;
          t.pad = (agroups << 8) | k;
          lst.push_back({(int64_t)t.count * (rows + 4) + (k == 0 && t.start == 0 ? D.n_skel : 0), t});
        }
        ++agroups;
      }
      // a block is split in every one of its column tiles or in none
      for (auto &x : lst) {
        const DevBlock &D = blocks[x.second.blk];
        if (D.pad2 > 1 && x.second.pad < 0 && x.second.count > 0) return fail(MHT_ERR_FORMAT, "adjoint split tiling");
      }
      std::stable_sort(lst.begin(), lst.end(), by_cost);
      P->adj[s] = Range{(int32_t)adj_all.size(), (int32_t)lst.size()};
      for (auto &x : lst) adj_all.push_back(x.second);
    }
    // multi-RHS adjoint K splits: on a stage with too few 64-column tiles to
    // fill the GPU several times over, a tile of a tall block would run one
    // long K loop; its rows are split into chunks of >= MMA_MIN_SPLIT (slabs
    // summed in order by the last CTA of the group).
    {
      const int nt = (int)amt[s].size();
      std::vector<std::pair<int64_t, Tile>> lst;
      for (auto &x : amt[s]) {
        DevBlock &D = blocks[x.second.blk];
        int ks = 1;
        if (nt > 0 && nt < MMA_TARGET && x.second.count > 0 && D.r_out >= 2 * MMA_MIN_SPLIT)
          ks = std::min(16, D.r_out / MMA_MIN_SPLIT);
        if (ks <= 1) {
          lst.push_back(x);
          continue;
        }
        if (D.mks == 0) {
          D.mks = ks;
          D.msp_off = mslabs;
          mslabs += (int64_t)((D.n_red + MMA_COLS - 1) / MMA_COLS) * ks;
        }
        const int bk = P->cplx ? 16 : 32;
        const int chunk = ((D.r_out + ks - 1) / ks + bk - 1) / bk * bk;
        for (int k = 0; k < ks; ++k) {
          const int rows = std::max(0, std::min(D.r_out, (k + 1) * chunk) - k * chunk);
          Tile t = x.second;
          t.pad = (mgroups << 8) | k;
          lst.push_back({(int64_t)t.count * (rows + 4) + (k == 0 && t.start == 0 ? D.n_skel : 0), t});
        }
        ++mgroups;
      }
      std::stable_sort(lst.begin(), lst.end(), by_cost);
      P->adjm[s] = Range{(int32_t)adjm_all.size(), (int32_t)lst.size()};
      for (auto &x : lst) adjm_all.push_back(x.second);
    }
  }

  // ------------------------------------------------ nrhs = 1 forward split-K
  // A stage with fewer than FWD1_TARGET row tiles leaves SMs idle; split the
  // columns of its blocks (>= FWD1_MIN_SPLIT columns per split) to reach the target.
  const int FWD1_TARGET = prop.multiProcessorCount * 6;
  const int FWD1_MIN_SPLIT = 64;  // columns per split
  std::vector<Tile> fwd1_all;
  P->fwd1.assign(L + 2, Range{});
  int64_t split_scalars = 0;
  int32_t groups = 0;
  for (int s = 0; s < L + 2; ++s) {
    const int nt = (int)ft[s].size();
    std::vector<std::pair<int64_t, Tile>> lst;
    for (auto &x : ft[s]) {
      DevBlock &D = blocks[x.second.blk];
      int ks = 1;
      if (nt > 0 && nt < FWD1_TARGET && D.n_red >= 2 * FWD1_MIN_SPLIT) {
        ks = (FWD1_TARGET + nt - 1) / nt;
        ks = std::min(ks, D.n_red / FWD1_MIN_SPLIT);
        ks = std::min(ks, 255);
      }
      if (ks <= 1) {
        lst.push_back(x);
        continue;
      }
      if (D.pad == 0) {  // first row tile of the block: reserve its scratch
        D.pad = ks;        // same split count for every row tile of the block
        D.fsp_off = split_scalars;
        split_scalars += (int64_t)((D.r_out + FWD_ROWS - 1) / FWD_ROWS) * ks * FWD_ROWS;
      }
    }
    for (auto &x : ft[s]) {
      const DevBlock &D = blocks[x.second.blk];
      if (D.pad <= 1) continue;
      const int ks = D.pad;
      const int chunk = ((D.n_red + ks - 1) / ks + 31) & ~31;
      for (int k = 0; k < ks; ++k) {
        const int cols = std::max(0, std::min(D.n_red, (k + 1) * chunk) - k * chunk);
        Tile t = x.second;
        t.pad = (groups << 8) | k;
        lst.push_back({(int64_t)t.count * (cols + 4), t});
      }
      ++groups;
    }
    std::stable_sort(lst.begin(), lst.end(), by_cost);
    P->fwd1[s] = Range{(int32_t)fwd1_all.size(), (int32_t)lst.size()};
    for (auto &x : lst) fwd1_all.push_back(x.second);
  }
  P->fwd1_lat.assign(L + 2, 0);
  for (int s = 0; s < L + 2; ++s) P->fwd1_lat[s] = P->fwd1[s].count < 2 * 7 * prop.multiProcessorCount ? 1 : 0;
  P->n_split_groups = groups;
  P->m_slabs = mslabs;
  P->m_groups = mgroups;

  // ------------------------------------------------ adjoint group-sum pieces
  // Readers: every materialised block's input segments.  For a source range
  // (c or a producer's zpool slot) the adjoint input is the sum of all reader
  // partials that cover it.
  struct Rd {
    int32_t src;
    int64_t start, len, pstart;
  };
  std::vector<Rd> readers;
  for (const DevBlock &D : blocks) {
    if (D.seg_len[0] > 0) readers.push_back({D.seg_src[0], D.seg_off[0], D.seg_len[0], D.part_off});
    if (D.seg_len[1] > 0) readers.push_back({D.seg_src[1], D.seg_off[1], D.seg_len[1], D.part_off + D.seg_len[0]});
  }
  // Fused group sums: a zpool producer whose output range is covered only by
  // readers that contain it whole gets the list of their partial offsets (in
  // reader-id order, the order reduce_kernel sums in); its consumer then sums
  // them on load and no reduction pass runs for it.
  std::vector<char> unfusable(blocks.size(), 0);
  std::vector<std::vector<int64_t>> rdl(blocks.size());
  {
    std::map<int64_t, int> prod_at;  // zpool out_off -> producer block
    for (int i = 0; i < (int)blocks.size(); ++i)
      if (!(blocks[i].flags & F_OUT_F) && blocks[i].r_out > 0) prod_at[blocks[i].out_off] = i;
    for (const Rd &r : readers) {
      if (r.src != SRC_Z) continue;
      auto it = prod_at.lower_bound(r.start);  // first producer starting at or after the reader
      if (it != prod_at.begin()) {              // a producer straddling the reader's start
        auto pv = std::prev(it);
        if (r.start < pv->first + blocks[pv->second].r_out) unfusable[pv->second] = 1;
      }
      for (; it != prod_at.end() && it->first < r.start + r.len; ++it) {
        if (it->first + blocks[it->second].r_out > r.start + r.len) unfusable[it->second] = 1;
        else rdl[it->second].push_back(r.pstart + (it->first - r.start));
      }
    }
  }
  // producer regions: c = [0, m) ("stage -1"), zpool slots of stage s <= L
  struct Region {
    int32_t src, stage;
    int64_t start, len;
    int blk;  // producer block (-1: the user's c)
    int32_t remote = 0;  // receive-buffer region: 1 + the sending rank
  };
  std::vector<Region> regions;
  if (!sharded) {
    regions.push_back({SRC_C, -1, 0, P->m, -1});
  } else {  // a shard owns (and writes in the adjoint) only its frequency leaves' slice of c
    const int64_t v0 = (int64_t)sh.g * (nl / sh.G), v1 = v0 + nl / sh.G;
    if (fr_off[v1] > fr_off[v0]) regions.push_back({SRC_C, -1, fr_off[v0], fr_off[v1] - fr_off[v0], -1});
  }
  for (int i = 0; i < (int)blocks.size(); ++i) {
    const DevBlock &D = blocks[i];
    // sharded: the switch stage's outputs (the send buffer) are read remotely;
    // their adjoint input arrives by the reverse exchange, no local sums
    if (sharded && block_stage[i] == sh.ls) continue;
    if (!(D.flags & F_OUT_F) && D.r_out > 0) regions.push_back({SRC_Z, block_stage[i], D.out_off, D.r_out, i});
  }
  // the receive buffer is a producer region of stage ls without a local
  // producer block: its adjoint sums are formed here and sent back
  for (const RecvRegion &rr : recv_regions)
    if (rr.len > 0) regions.push_back({SRC_Z, sh.ls, rr.off, rr.len, -1, rr.src + 1});
  std::vector<std::vector<Piece>> pcs(L + 3);  // index stage+1 (0 = c)
  std::vector<std::vector<std::vector<int64_t>>> pcs_rd(L + 3);
  std::vector<std::vector<char>> pcs_keep(L + 3);  // piece still needed in fused mode
  for (int src : {SRC_C, SRC_Z}) {
    std::vector<int64_t> cuts;
    std::vector<const Region *> regs;
    for (const Region &g : regions)
      if (g.src == src) {
        regs.push_back(&g);
        cuts.push_back(g.start);
        cuts.push_back(g.start + g.len);
      }
    std::vector<int> rids;
    for (int i = 0; i < (int)readers.size(); ++i)
      if (readers[i].src == src) {
        rids.push_back(i);
        cuts.push_back(readers[i].start);
        cuts.push_back(readers[i].start + readers[i].len);
      }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    std::sort(regs.begin(), regs.end(), [](const Region *a, const Region *b) { return a->start < b->start; });
    // events sorted by coordinate
    std::vector<std::pair<int64_t, int>> starts, ends;
    for (int i : rids) {
      starts.push_back({readers[i].start, i});
      ends.push_back({readers[i].start + readers[i].len, i});
    }
    std::sort(starts.begin(), starts.end());
    std::sort(ends.begin(), ends.end());
    std::set<int> active;
    size_t si = 0, ei = 0, ri = 0;
    for (size_t k = 0; k + 1 < cuts.size(); ++k) {
      const int64_t a = cuts[k], e = cuts[k + 1];
      while (ei < ends.size() && ends[ei].first <= a) active.erase(ends[ei++].second);
      while (si < starts.size() && starts[si].first <= a) {
        if (readers[starts[si].second].start + readers[starts[si].second].len > a) active.insert(starts[si].second);
        ++si;
      }
      while (ri < regs.size() && regs[ri]->start + regs[ri]->len <= a) ++ri;
      if (ri >= regs.size() || regs[ri]->start > a) {
        if (!active.empty()) return fail(MHT_ERR_FORMAT, "reader outside any producer region");
        continue;
      }
      const int slot = regs[ri]->stage + 1;
      for (int64_t c0 = a; c0 < e; c0 += 1024) {
        Piece pc;
        memset(&pc, 0, sizeof pc);
        pc.dst_src = src;
        pc.dst_off = c0;
        pc.remote = regs[ri]->remote;
        pc.len = (int32_t)std::min<int64_t>(1024, e - c0);
        std::vector<int64_t> rr;
        for (int id : active) rr.push_back(readers[id].pstart + (c0 - readers[id].start));
        pc.rd_count = (int32_t)rr.size();
        pcs[slot].push_back(pc);
        pcs_rd[slot].push_back(std::move(rr));
        pcs_keep[slot].push_back(regs[ri]->blk < 0 || unfusable[regs[ri]->blk]);
      }
    }
  }
  std::vector<Piece> pieces_all;
  std::vector<int64_t> rd_all;
  P->pieces.assign(L + 2, Range{});
  P->pieces_u.assign(L + 2, Range{});
  for (int slot = 0; slot < L + 3; ++slot) {
    // all pieces of the slot (unfused mode), then the unfused producers' pieces
    // again as their own range (fused mode)
    for (int pass = 0; pass < (slot == 0 ? 1 : 2); ++pass) {
      Range rg{(int32_t)pieces_all.size(), 0};
      for (size_t k = 0; k < pcs[slot].size(); ++k) {
        if (pass == 1 && !pcs_keep[slot][k]) continue;
        Piece pc = pcs[slot][k];
        pc.rd_begin = (int64_t)rd_all.size();
        rd_all.insert(rd_all.end(), pcs_rd[slot][k].begin(), pcs_rd[slot][k].end());
        pieces_all.push_back(pc);
        ++rg.count;
      }
      if (slot == 0)
        P->cpieces = rg;
      else if (pass == 0)
        P->pieces[slot - 1] = rg;
      else
        P->pieces_u[slot - 1] = rg;
    }
  }
  // per-block fused reader lists
  std::vector<int64_t> rdtab;
  P->n_unfused = 0;
  for (int i = 0; i < (int)blocks.size(); ++i)
    if (sharded && block_stage[i] == sh.ls) unfusable[i] = 1;  // input arrives by the exchange
  for (int i = 0; i < (int)blocks.size(); ++i) {
    DevBlock &D = blocks[i];
    D.rd_off = (int64_t)rdtab.size();
    if (D.flags & F_OUT_F) {
      D.rd_cnt = 0;
    } else if (unfusable[i]) {
      D.rd_cnt = -1;
      ++P->n_unfused;
    } else {
      D.rd_cnt = (int32_t)rdl[i].size();
      rdtab.insert(rdtab.end(), rdl[i].begin(), rdl[i].end());
    }
  }

  // ------------------------------------------------ upload
  mht_status st;
  if ((st = upload(&P->d_idx, idx_all, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_perm, perm, P->device_bytes)) != MHT_OK) return st;
  if (!perm_k.empty() && (st = upload(&P->d_permk, perm_k, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_blocks, blocks, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_fwd, fwd_all, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_fwd1, fwd1_all, P->device_bytes)) != MHT_OK) return st;
  // split scratch + arrival counters, shared by the forward (row tiles split
  // by columns) and the adjoint (column tiles split by rows): applies on one
  // plan are serialised on its stream, and the last CTA of a group re-arms
  // its counter
  const int64_t sp_scalars = std::max<int64_t>({split_scalars, asplit_scalars, 1});
  const int64_t sp_groups = std::max<int64_t>({(int64_t)groups, (int64_t)agroups, 1});
  CUDA_TRY(cudaMalloc(&P->d_fsplit, (size_t)sp_scalars * P->ssz));
  CUDA_TRY(cudaMalloc((void **)&P->d_fcount, (size_t)sp_groups * sizeof(int)));
  CUDA_TRY(cudaMemset(P->d_fcount, 0, (size_t)sp_groups * sizeof(int)));
  P->device_bytes += sp_scalars * (int64_t)P->ssz + sp_groups * 4;
  if ((st = upload(&P->d_adj, adj_all, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_adjm, adjm_all, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_pieces, pieces_all, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_rd, rd_all, P->device_bytes)) != MHT_OK) return st;
  if ((st = upload(&P->d_rdtab, rdtab, P->device_bytes)) != MHT_OK) return st;
  return MHT_OK;
}

mht_status ensure_ws(mht_plan *P, int nrhs) {
  if (nrhs <= P->ws_nrhs) return MHT_OK;
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->clear_graphs();
  if (P->d_z) cudaFree(P->d_z);
  if (P->d_part) cudaFree(P->d_part);
  P->d_z = P->d_part = nullptr;
  P->ws_nrhs = 0;
  if (P->x_on) return fail(MHT_ERR_INVALID_ARG, "fused exchange set up for a smaller nrhs: mht_shard_close_peers first");
  // sharded plans: the fused exchange's sync area after the workspace (zeroed)
  P->sync_byte_off = ((int64_t)P->Zt * nrhs * (int64_t)P->ssz + 255) / 256 * 256;
  const size_t sync_bytes = P->shard_G > 1 ? (size_t)(2 * P->shard_G + 2) * 8 : 0;
  CUDA_TRY(cudaMalloc(&P->d_z, (size_t)P->sync_byte_off + sync_bytes));
  if (sync_bytes) CUDA_TRY(cudaMemset(static_cast<char *>(P->d_z) + P->sync_byte_off, 0, sync_bytes));
  CUDA_TRY(cudaMalloc(&P->d_part, (size_t)P->Pt * nrhs * P->ssz));
  if (P->d_msplit) cudaFree(P->d_msplit);
  if (P->d_mcount) cudaFree(P->d_mcount);
  P->d_msplit = nullptr;
  P->d_mcount = nullptr;
  CUDA_TRY(cudaMalloc(&P->d_msplit, (size_t)std::max<int64_t>(1, P->m_slabs * MMA_COLS * nrhs) * P->ssz));
  const size_t ncnt = (size_t)std::max<int64_t>(1, (int64_t)P->m_groups * ((nrhs + 7) / 8));
  CUDA_TRY(cudaMalloc((void **)&P->d_mcount, ncnt * sizeof(int)));
  CUDA_TRY(cudaMemset(P->d_mcount, 0, ncnt * sizeof(int)));
  P->ws_nrhs = nrhs;
  return MHT_OK;
}

Ctx make_ctx(mht_plan *P, int nrhs) {
  Ctx cx;
  memset(&cx, 0, sizeof cx);
  cx.coef = P->d_coef;
  cx.idx = P->d_idx;
  cx.perm = P->d_perm;
  cx.permk = P->d_permk;
  cx.blocks = P->d_blocks;
  cx.z = P->d_z;
  cx.part = P->d_part;
  cx.fsplit = P->d_fsplit;
  cx.fcount = P->d_fcount;
  cx.rdtab = P->d_rdtab;
  cx.tmaps = P->d_tmaps;
  cx.diag = P->cur_diag;
  cx.diag_sqrt = P->cur_diag_sqrt;
  cx.msplit = P->d_msplit;
  cx.mcount = P->d_mcount;
  // fused group sums only at nrhs = 1: the multi-RHS gathers measured faster
  // from the reduced workspace (profiles/r01_fused_sums_ab.txt)
  cx.fused = (P->fused_sum && nrhs == 1) ? 1 : 0;
  cx.m = P->m;
  cx.n = P->n;
  cx.Zt = P->Zt;
  cx.Pt = P->Pt;
  cx.nrhs = nrhs;
  if (P->x_on) {
    cx.zrem = P->d_zrem;
    cx.zdel = P->d_zdel;
    cx.zG = P->shard_G;
  }
  return cx;
}

cudaEvent_t next_event(mht_plan *P) {
  if (P->ev_used == P->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    P->ev_pool.push_back(e);
  }
  return P->ev_pool[P->ev_used++];
}

// Launch wrapper: brackets the launch with events when profiling is on.
template <class F>
void timed(mht_plan *P, int kind, int stage, int nrhs, int count, F &&launch) {
  if (count <= 0) return;
  if (!P->prof) {
    launch();
    return;
  }
  cudaEvent_t a = next_event(P), b = next_event(P);
  if (!a || !b) {
    launch();
    return;
  }
  cudaEventRecord(a, P->stream);
  launch();
  cudaEventRecord(b, P->stream);
  P->recs.push_back({kind, stage, nrhs, a, b});
}

// part: 0 the whole apply; sharded plans 1 = stages 0..ls (before the
// exchange), 2 = stages ls+1..L+1 (after it)
mht_status run_forward(mht_plan *P, const void *c, void *f, int nrhs, int part = 0) {
  Ctx cx = make_ctx(P, nrhs);
  cx.c = c;
  cx.fout = f;
  const int s_lo = part == 2 ? P->shard_ls + 1 : 0, s_hi = part == 1 ? P->shard_ls : P->L + 1;
  unsigned long long *own_sync =
      reinterpret_cast<unsigned long long *>(static_cast<char *>(P->d_z) + P->sync_byte_off);
  if (part == 2 && P->x_on) launch_xwait(own_sync, 0, P->shard_G, P->stream);  // every peer's z_ls stores landed
  for (int s = s_lo; s <= s_hi; ++s)
    timed(P, 0, s, nrhs, nrhs == 1 ? P->fwd1[s].count : P->fwd[s].count, [&] {
      if (nrhs == 1)
        launch_fwd(P->cplx, cx, P->d_fwd1 + P->fwd1[s].off, P->fwd1[s].count, P->fwd1_lat[s] != 0, P->stream);
      else
        launch_mma(P->cplx, false, cx, P->d_fwd + P->fwd[s].off, P->fwd[s].count, false, P->stream);
    });
  if (part == 1 && P->x_on) launch_xsignal(own_sync, P->d_peersync, 0, P->shard_g, P->shard_G, P->stream);
  CUDA_TRY(cudaGetLastError());
  return MHT_OK;
}

// part: 0 the whole adjoint; sharded plans 1 = leaf stage .. ls+1 plus the
// sums into the receive buffer (sent back by the reverse exchange), 2 = stage
// ls (its input arrived) .. 0 plus the sums into c
mht_status run_adjoint(mht_plan *P, const void *f, void *c, int nrhs, int part = 0) {
  Ctx cx = make_ctx(P, nrhs);
  cx.fin = f;
  cx.cw = c;
  const int L = P->L;
  auto adj_stage = [&](int s, bool from_f) {
    if (nrhs == 1)
      timed(P, 1, s, nrhs, P->adj[s].count,
            [&] { launch_adj(P->cplx, cx, P->d_adj + P->adj[s].off, P->adj[s].count, from_f, P->stream); });
    else
      timed(P, 1, s, nrhs, P->adjm[s].count, [&] {
        launch_mma(P->cplx, true, cx, P->d_adjm + P->adjm[s].off, P->adjm[s].count, from_f, P->stream);
      });
  };
  auto sums = [&](int s) {
    const Range pr = cx.fused ? P->pieces_u[s] : P->pieces[s];
    timed(P, 2, s, nrhs, pr.count, [&] {
      launch_reduce(P->cplx, cx, P->d_pieces + pr.off, P->d_rd, pr.count, P->stream);
    });
  };
  const int ls = P->shard_ls;
  unsigned long long *own_sync =
      reinterpret_cast<unsigned long long *>(static_cast<char *>(P->d_z) + P->sync_byte_off);
  if (part != 2) {
    adj_stage(L + 1, true);
    for (int s = L; s >= (part == 1 ? ls + 1 : 0); --s) {
      sums(s);
      adj_stage(s, false);
    }
    if (part == 1) sums(ls);
    if (part == 1 && P->x_on) launch_xsignal(own_sync, P->d_peersync, 1, P->shard_g, P->shard_G, P->stream);
  }
  if (part == 2) {
    if (P->x_on) launch_xwait(own_sync, 1, P->shard_G, P->stream);  // the peers' sums landed in the send buffer
    adj_stage(ls, false);
    for (int s = ls - 1; s >= 0; --s) {
      sums(s);
      adj_stage(s, false);
    }
  }
  if (part != 1)
    timed(P, 2, -1, nrhs, P->cpieces.count, [&] {
      launch_reduce(P->cplx, cx, P->d_pieces + P->cpieces.off, P->d_rd, P->cpieces.count, P->stream);
    });
  CUDA_TRY(cudaGetLastError());
  return MHT_OK;
}

// Replay (or capture, then replay) the whole stage sequence of one apply as a
// CUDA graph.  Profiling bypasses graphs (per-launch events).
// dir: 0 synthesis, 1 analysis; sharded halves 2 / 3 synthesis before / after
// the exchange, 4 / 5 analysis before / after the reverse exchange
mht_status run_seq(mht_plan *P, int dir, const void *src, void *dst, int nrhs) {
  switch (dir) {
    case 0: return run_forward(P, src, dst, nrhs);
    case 1: return run_adjoint(P, src, dst, nrhs);
    case 2: return run_forward(P, src, nullptr, nrhs, 1);
    case 3: return run_forward(P, nullptr, dst, nrhs, 2);
    case 4: return run_adjoint(P, src, nullptr, nrhs, 1);
    default: return run_adjoint(P, nullptr, dst, nrhs, 2);
  }
}

mht_status run_dir(mht_plan *P, int dir, const void *src, void *dst, int nrhs) {
  if (!P->graphs || P->prof) return run_seq(P, dir, src, dst, nrhs);
  mht_plan::GraphKey key{dir, nrhs, src, dst, P->cur_diag, P->cur_diag_sqrt};
  auto it = P->gcache.find(key);
  if (it == P->gcache.end()) {
    if (!P->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&P->cap_stream, cudaStreamNonBlocking));
    if (P->gcache.size() >= 32) P->clear_graphs();
    cudaStream_t user = P->stream;
    P->stream = P->cap_stream;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal);
    mht_status st = MHT_OK;
    if (e == cudaSuccess) {
      st = run_seq(P, dir, src, dst, nrhs);
      e = cudaStreamEndCapture(P->cap_stream, &g);
    }
    P->stream = user;
    if (st != MHT_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return fail(MHT_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(MHT_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    it = P->gcache.emplace(key, ex).first;
  }
  CUDA_TRY(cudaGraphLaunch(it->second, P->stream));
  return MHT_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

mht_status mht_plan_load(const char *path, int device, mht_plan **out) {
  if (!path || !out) return fail(MHT_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  try {
    std::unique_ptr<mht_plan> P(new mht_plan());
    mht_status s = load_impl(path, device, P, ShardCfg());
    if (s != MHT_OK) return s;
    *out = P.release();
    return MHT_OK;
  } catch (const std::bad_alloc &) {
    return fail(MHT_ERR_OOM, "host allocation failed");
  } catch (...) {
    return fail(MHT_ERR_CUDA, "unexpected exception in loader");
  }
}

mht_status mht_plan_load_shard(const char *path, int device, int nshards, int shard, int switch_level,
                               mht_plan **out) {
  if (!path || !out || nshards < 1 || shard < 0 || shard >= nshards || (nshards & (nshards - 1)) != 0)
    return fail(MHT_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  try {
    std::unique_ptr<mht_plan> P(new mht_plan());
    ShardCfg sh;
    sh.G = nshards;
    sh.g = shard;
    sh.ls = switch_level;
    if (nshards > 1) {
      // L is needed to place / check the switch level: peek at the header
      FILE *fp = fopen(path, "rb");
      if (!fp) return fail(MHT_ERR_IO, std::string("cannot open ") + path);
      unsigned char hdr[256];
      const size_t got = fread(hdr, 1, 256, fp);
      fclose(fp);
      if (got != 256 || memcmp(hdr, "BFMHTPLN", 8) != 0) return fail(MHT_ERR_FORMAT, "bad header");
      int32_t L;
      memcpy(&L, hdr + 32, 4);
      int lg = 0;
      while ((1 << lg) < nshards) ++lg;
      if (sh.ls < 0) sh.ls = std::max(lg, L / 2);
      if (L < 2 * lg || sh.ls < lg || sh.ls > L - lg)
        return fail(MHT_ERR_INVALID_ARG, "switch level must satisfy log2 G <= ls <= L - log2 G");
    }
    mht_status s = load_impl(path, device, P, sh);
    if (s != MHT_OK) return s;
    *out = P.release();
    return MHT_OK;
  } catch (const std::bad_alloc &) {
    return fail(MHT_ERR_OOM, "host allocation failed");
  } catch (...) {
    return fail(MHT_ERR_CUDA, "unexpected exception in loader");
  }
}

mht_status mht_shard_info(const mht_plan *P, int32_t *nshards, int32_t *shard, int32_t *switch_level,
                          int64_t *send_off, int64_t *send_len, int64_t *recv_off, int64_t *recv_len) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  if (nshards) *nshards = P->shard_G;
  if (shard) *shard = P->shard_g;
  if (switch_level) *switch_level = P->shard_ls;
  for (int h = 0; h < (int)P->send_off.size(); ++h) {
    if (send_off) send_off[h] = P->send_off[h];
    if (send_len) send_len[h] = P->send_len[h];
    if (recv_off) recv_off[h] = P->recv_off[h];
    if (recv_len) recv_len[h] = P->recv_len[h];
  }
  return MHT_OK;
}

mht_status mht_shard_workspace(mht_plan *P, int nrhs, void **zpool) {
  if (!P || !zpool || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  *zpool = P->d_z;
  return MHT_OK;
}

static mht_status shard_call(mht_plan *P, int dir, const void *src, void *dst, int nrhs) {
  if (!P || nrhs < 1 || (!src && !dst)) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G < 2) return fail(MHT_ERR_INVALID_ARG, "not a sharded plan (mht_plan_load_shard with nshards > 1)");
  if (P->x_on && nrhs > P->x_nrhs) return fail(MHT_ERR_INVALID_ARG, "nrhs above the fused exchange's set-up width");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  return run_dir(P, dir, src, dst, nrhs);
}

mht_status mht_shard_export(mht_plan *P, int nrhs, void *ipc_handle, int64_t *layout) {
  if (!P || nrhs < 1 || !layout) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G < 2) return fail(MHT_ERR_INVALID_ARG, "not a sharded plan (mht_plan_load_shard with nshards > 1)");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, P->d_z));
    memcpy(ipc_handle, &h, sizeof h);
  }
  const int G = P->shard_G;
  for (int h = 0; h < G; ++h) {
    layout[h] = P->recv_off[h];
    layout[G + h] = P->send_off[h];
  }
  layout[2 * G] = P->sync_byte_off;
  return MHT_OK;
}

mht_status mht_shard_set_peers(mht_plan *P, int nrhs, void *const *bases, const int64_t *layouts) {
  if (!P || nrhs < 1 || !bases || !layouts) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G < 2) return fail(MHT_ERR_INVALID_ARG, "not a sharded plan (mht_plan_load_shard with nshards > 1)");
  const int G = P->shard_G, g = P->shard_g, LW = 2 * G + 1;
  if (P->x_on && nrhs != P->x_nrhs) return fail(MHT_ERR_INVALID_ARG, "fused exchange already set up for another nrhs");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  if (bases[g] != P->d_z) return fail(MHT_ERR_INVALID_ARG, "bases[shard] must be this plan's own workspace");
  for (int h = 0; h < G; ++h) {
    if (!bases[h]) return fail(MHT_ERR_INVALID_ARG, "null peer base");
    const int64_t *lh = layouts + (int64_t)h * LW;
    // every rank's layout is its own; the exchange is only consistent if the
    // pair (g -> h) agrees on the block count: checked through the lengths
    if (lh[g] < 0 || lh[G + g] < 0) return fail(MHT_ERR_INVALID_ARG, "bad peer layout");
  }
  std::vector<void *> zrem(2 * G);
  std::vector<int64_t> zdel(2 * G);
  std::vector<unsigned long long *> psync(G);
  for (int h = 0; h < G; ++h) {
    const int64_t *lh = layouts + (int64_t)h * LW;
    // forward: my send region for h -> h's receive region from me
    zrem[h] = bases[h];
    zdel[h] = lh[g] - P->send_off[h];
    // adjoint: my receive region from h -> h's send region for me
    zrem[G + h] = bases[h];
    zdel[G + h] = lh[G + g] - P->recv_off[h];
    psync[h] = reinterpret_cast<unsigned long long *>(static_cast<char *>(bases[h]) + lh[2 * G]);
  }
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->clear_graphs();
  if (!P->d_zrem) {
    CUDA_TRY(cudaMalloc((void **)&P->d_zrem, 2 * G * sizeof(void *)));
    CUDA_TRY(cudaMalloc((void **)&P->d_zdel, 2 * G * sizeof(int64_t)));
    CUDA_TRY(cudaMalloc((void **)&P->d_peersync, G * sizeof(void *)));
  }
  CUDA_TRY(cudaMemcpy(P->d_zrem, zrem.data(), 2 * G * sizeof(void *), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->d_zdel, zdel.data(), 2 * G * sizeof(int64_t), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->d_peersync, psync.data(), G * sizeof(void *), cudaMemcpyHostToDevice));
  P->x_on = true;
  P->x_nrhs = nrhs;
  return MHT_OK;
}

mht_status mht_shard_open_peers(mht_plan *P, int nrhs, const void *ipc_handles, const int64_t *layouts) {
  if (!P || nrhs < 1 || !ipc_handles || !layouts) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G < 2) return fail(MHT_ERR_INVALID_ARG, "not a sharded plan (mht_plan_load_shard with nshards > 1)");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  const int G = P->shard_G;
  std::vector<void *> bases(G, nullptr);
  for (int h = 0; h < G; ++h) {
    if (h == P->shard_g) {
      bases[h] = P->d_z;
      continue;
    }
    cudaIpcMemHandle_t hd;
    memcpy(&hd, static_cast<const char *>(ipc_handles) + (size_t)h * sizeof hd, sizeof hd);
    void *ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    P->ipc_open.push_back(ptr);
    bases[h] = ptr;
  }
  return mht_shard_set_peers(P, nrhs, bases.data(), layouts);
}

mht_status mht_shard_close_peers(mht_plan *P) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->clear_graphs();
  P->x_on = false;
  P->x_nrhs = 0;
  for (void *q : P->ipc_open) cudaIpcCloseMemHandle(q);
  P->ipc_open.clear();
  return MHT_OK;
}

mht_status mht_apply_shard_begin(mht_plan *P, const void *c, int nrhs) { return shard_call(P, 2, c, nullptr, nrhs); }
mht_status mht_apply_shard_end(mht_plan *P, void *f, int nrhs) { return shard_call(P, 3, nullptr, f, nrhs); }
mht_status mht_apply_adjoint_shard_begin(mht_plan *P, const void *f, int nrhs) {
  return shard_call(P, 4, f, nullptr, nrhs);
}
mht_status mht_apply_adjoint_shard_end(mht_plan *P, void *c, int nrhs) { return shard_call(P, 5, nullptr, c, nrhs); }

mht_status mht_plan_info_get(const mht_plan *P, mht_plan_info *info) {
  if (!P || !info) return fail(MHT_ERR_INVALID_ARG, "null argument");
  memset(info, 0, sizeof *info);
  info->n = P->n;
  info->m = P->m;
  info->L = P->L;
  info->dtype = P->cplx ? MHT_DTYPE_C128 : MHT_DTYPE_F64;
  info->tol = P->tol;
  info->plan_bytes = P->plan_bytes;
  info->factor_entries = P->factor_entries;
  info->device_bytes = P->device_bytes;
  info->index_entries = P->index_entries;
  info->n_materialized = P->n_mat;
  info->n_alias = P->n_alias;
  int f = 0, a = 0;
  for (int s = 0; s < P->L + 2; ++s) {
    f += P->fwd[s].count > 0;
    a += (P->adj[s].count > 0) + (s <= P->L && (P->fused_sum ? P->pieces_u[s] : P->pieces[s]).count > 0);
  }
  a += P->cpieces.count > 0;
  info->fwd_launches = f;
  info->adj_launches = a;
  return MHT_OK;
}

mht_status mht_plan_set_stream(mht_plan *P, void *stream) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  // applies go to the caller's stream; the plan's own stream (used by the
  // loader, and again after mht_plan_set_stream(P, own)) is kept and
  // destroyed with the plan.  Work already queued on the previous stream is
  // ordered before later calls by synchronising it first.
  CUDA_TRY(cudaSetDevice(P->device));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->stream = static_cast<cudaStream_t>(stream);
  return MHT_OK;
}

mht_status mht_reserve(mht_plan *P, int nrhs) {
  if (!P || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  CUDA_TRY(cudaSetDevice(P->device));
  return ensure_ws(P, nrhs);
}

mht_status mht_apply(mht_plan *P, const void *c, void *f, int nrhs) {
  if (!P || !c || !f || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use mht_apply_shard_begin / _end");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  return run_dir(P, 0, c, f, nrhs);
}

mht_status mht_apply_adjoint(mht_plan *P, const void *f, void *c, int nrhs) {
  if (!P || !c || !f || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use mht_apply_adjoint_shard_begin / _end");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  return run_dir(P, 1, f, c, nrhs);
}

namespace {
struct DiagScope {  // sets the plan's coefficient-side diagonal for one call
  mht_plan *P;
  DiagScope(mht_plan *p, const double *d, int sq) : P(p) {
    P->cur_diag = d;
    P->cur_diag_sqrt = sq;
  }
  ~DiagScope() {
    P->cur_diag = nullptr;
    P->cur_diag_sqrt = 0;
  }
};
}  // namespace

mht_status mht_apply_diag(mht_plan *P, const void *c, const double *d, void *f, int nrhs) {
  if (!P || !c || !d || !f || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  DiagScope ds(P, d, 0);
  return run_dir(P, 0, c, f, nrhs);
}

mht_status mht_apply_adjoint_diag(mht_plan *P, const void *f, const double *d, void *c, int nrhs) {
  if (!P || !c || !d || !f || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  DiagScope ds(P, d, 0);
  return run_dir(P, 1, f, c, nrhs);
}

mht_status mht_grf_sample(mht_plan *P, const void *z, const double *S, void *y, int nrhs) {
  if (!P || !z || !S || !y || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  DiagScope ds(P, S, 1);
  return run_dir(P, 0, z, y, nrhs);
}

mht_status mht_covariance_apply(mht_plan *P, const void *v, const double *S, void *out, int nrhs) {
  if (!P || !v || !S || !out || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s = ensure_ws(P, nrhs);
  if (s != MHT_OK) return s;
  if (nrhs > P->ctmp_nrhs) {
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    P->clear_graphs();
    if (P->d_ctmp) cudaFree(P->d_ctmp);
    P->d_ctmp = nullptr;
    P->ctmp_nrhs = 0;
    CUDA_TRY(cudaMalloc(&P->d_ctmp, (size_t)P->m * nrhs * P->ssz));
    P->ctmp_nrhs = nrhs;
  }
  {
    DiagScope ds(P, S, 0);  // c = S Phi^* v  (diagonal fused into the adjoint's final sums)
    if ((s = run_dir(P, 1, v, P->d_ctmp, nrhs)) != MHT_OK) return s;
  }
  return run_dir(P, 0, P->d_ctmp, out, nrhs);  // out = Phi c
}

// ---------------------------------------------------------------- LSQR
// Inverse MHT (§7.1, Eq. inverse-MHT): Paige &
// Saunders' LSQR on Phi, every iteration = one synthesis + one analysis of
// the plan plus the vector kernels of mht_lsqr.cu; per-column scalars stay on
// the device.  Convergence is checked every `check_every` iterations
// (one small device-to-host copy).
mht_status mht_lsqr(mht_plan *P, const void *b, void *x, int nrhs, int max_iters, double atol, double btol,
                    int *iters_done, double *rnorm, double *arnorm) {
  if (!P || !b || !x || nrhs < 1 || max_iters < 0) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status st = ensure_ws(P, nrhs);
  if (st != MHT_OK) return st;
  const int64_t n = P->n, m = P->m;
  const size_t sz = P->ssz;
  const int pn = lsqr_partials(n), pm = lsqr_partials(m);
  const int pmax = std::max(pn, pm);
  if (nrhs > P->lsqr_nrhs) {
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    P->clear_graphs();  // graphs keyed on the old work vectors
    for (void *&p : P->lsqr_buf) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    P->lsqr_nrhs = 0;
    const size_t bytes[7] = {(size_t)n * nrhs * sz, (size_t)m * nrhs * sz, (size_t)m * nrhs * sz, (size_t)n * nrhs * sz,
                             (size_t)m * nrhs * sz, (size_t)pmax * nrhs * sizeof(double), (size_t)nrhs * sizeof(LsqrCol)};
    for (int i = 0; i < 7; ++i) CUDA_TRY(cudaMalloc(&P->lsqr_buf[i], bytes[i]));
    P->lsqr_nrhs = nrhs;
  }
  struct Buf {
    void *p;
  } u{P->lsqr_buf[0]}, v{P->lsqr_buf[1]}, w{P->lsqr_buf[2]}, tn{P->lsqr_buf[3]}, tm{P->lsqr_buf[4]};
  CUDA_TRY(cudaMemsetAsync(P->lsqr_buf[6], 0, (size_t)nrhs * sizeof(LsqrCol), P->stream));
  LsqrCol *dc = static_cast<LsqrCol *>(P->lsqr_buf[6]);
  double *dp = static_cast<double *>(P->lsqr_buf[5]);
  void *s = P->stream;
  const bool cx = P->cplx;
  // beta_1 u_1 = b;  alpha_1 v_1 = Phi^* u_1;  w_1 = v_1;  x_0 = 0
  lsqr_axpy_norm(cx, b, u.p, n, nrhs, nullptr, 0, dp, s);
  lsqr_scalars(dp, pn, nrhs, dc, 2, s);
  lsqr_scale(cx, u.p, n, nrhs, dc, 0, s);
  if ((st = run_dir(P, 1, u.p, v.p, nrhs)) != MHT_OK) return st;
  lsqr_axpy_norm(cx, v.p, v.p, m, nrhs, nullptr, 0, dp, s);
  lsqr_scalars(dp, pm, nrhs, dc, 3, s);
  lsqr_update(cx, v.p, w.p, x, m, nrhs, dc, 1, s);
  CUDA_TRY(cudaGetLastError());
  const bool check = atol > 0 || btol > 0;
  const int every = 10;
  std::vector<LsqrCol> h(nrhs);
  int it = 0;
  for (; it < max_iters; ++it) {
    // beta u = Phi v - alpha u
    if ((st = run_dir(P, 0, v.p, tn.p, nrhs)) != MHT_OK) return st;
    lsqr_axpy_norm(cx, tn.p, u.p, n, nrhs, dc, 0, dp, s);
    lsqr_scalars(dp, pn, nrhs, dc, 0, s);
    lsqr_scale(cx, u.p, n, nrhs, dc, 0, s);
    // alpha v = Phi^* u - beta v, rotation, x / w updates
    if ((st = run_dir(P, 1, u.p, tm.p, nrhs)) != MHT_OK) return st;
    lsqr_axpy_norm(cx, tm.p, v.p, m, nrhs, dc, 1, dp, s);
    lsqr_scalars(dp, pm, nrhs, dc, 1, s);
    lsqr_update(cx, v.p, w.p, x, m, nrhs, dc, 0, s);
    if (check && ((it + 1) % every == 0 || it + 1 == max_iters)) {
      lsqr_xnorm(cx, x, m, nrhs, dp, dc, s);
      CUDA_TRY(cudaMemcpyAsync(h.data(), dc, (size_t)nrhs * sizeof(LsqrCol), cudaMemcpyDeviceToHost,
                               (cudaStream_t)s));
      CUDA_TRY(cudaStreamSynchronize((cudaStream_t)s));
      bool all = true;
      for (const LsqrCol &c : h) {
        const double an = sqrt(c.anorm2);
        const bool t1 = c.rnorm <= btol * c.bnorm + atol * an * c.xnorm;
        const bool t2 = c.arnorm <= atol * an * c.rnorm;
        all = all && (t1 || t2);
      }
      if (all) {
        ++it;
        break;
      }
    }
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(h.data(), dc, (size_t)nrhs * sizeof(LsqrCol), cudaMemcpyDeviceToHost, (cudaStream_t)s));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)s));
  if (iters_done) *iters_done = it;
  for (int r = 0; r < nrhs; ++r) {
    if (rnorm) rnorm[r] = h[r].rnorm;
    if (arnorm) arnorm[r] = h[r].arnorm;
  }
  return MHT_OK;
}

static mht_status ensure_host_staging(mht_plan *P, int nrhs) {
  if (nrhs <= P->host_nrhs) return MHT_OK;
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->clear_graphs();
  if (P->d_hc) cudaFree(P->d_hc);
  if (P->d_hf) cudaFree(P->d_hf);
  P->d_hc = P->d_hf = nullptr;
  P->host_nrhs = 0;
  CUDA_TRY(cudaMalloc(&P->d_hc, (size_t)P->m * nrhs * P->ssz));
  CUDA_TRY(cudaMalloc(&P->d_hf, (size_t)P->n * nrhs * P->ssz));
  P->host_nrhs = nrhs;
  return MHT_OK;
}

mht_status mht_apply_host(mht_plan *P, const void *c_host, void *f_host, int nrhs) {
  if (!P || !c_host || !f_host || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s;
  if ((s = ensure_ws(P, nrhs)) != MHT_OK || (s = ensure_host_staging(P, nrhs)) != MHT_OK) return s;
  CUDA_TRY(cudaMemcpyAsync(P->d_hc, c_host, (size_t)P->m * nrhs * P->ssz, cudaMemcpyHostToDevice, P->stream));
  if ((s = run_dir(P, 0, P->d_hc, P->d_hf, nrhs)) != MHT_OK) return s;
  CUDA_TRY(cudaMemcpyAsync(f_host, P->d_hf, (size_t)P->n * nrhs * P->ssz, cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  return MHT_OK;
}

mht_status mht_apply_adjoint_host(mht_plan *P, const void *f_host, void *c_host, int nrhs) {
  if (!P || !c_host || !f_host || nrhs < 1) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status s;
  if ((s = ensure_ws(P, nrhs)) != MHT_OK || (s = ensure_host_staging(P, nrhs)) != MHT_OK) return s;
  CUDA_TRY(cudaMemcpyAsync(P->d_hf, f_host, (size_t)P->n * nrhs * P->ssz, cudaMemcpyHostToDevice, P->stream));
  if ((s = run_dir(P, 1, P->d_hf, P->d_hc, nrhs)) != MHT_OK) return s;
  CUDA_TRY(cudaMemcpyAsync(c_host, P->d_hc, (size_t)P->m * nrhs * P->ssz, cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  return MHT_OK;
}

// Batch of independent host-buffer transforms, pipelined: job i's input copy
// (stream s_in) overlaps job i-1's transform (the plan's stream) and job i-2's
// output copy (stream s_out); two staging slots, ordered by events.
mht_status mht_apply_host_batch(mht_plan *P, const mht_host_job *jobs, int njobs) {
  if (!P || (njobs > 0 && !jobs) || njobs < 0) return fail(MHT_ERR_INVALID_ARG, "bad argument");
  if (P->shard_G > 1) return fail(MHT_ERR_INVALID_ARG, "sharded plan: use the mht_*_shard_* calls");
  int maxr = 0;
  for (int i = 0; i < njobs; ++i) {
    const mht_host_job &J = jobs[i];
    if ((J.dir != 0 && J.dir != 1) || J.nrhs < 1 || !J.in || !J.out) return fail(MHT_ERR_INVALID_ARG, "bad job");
    maxr = std::max(maxr, J.nrhs);
  }
  if (njobs == 0) return MHT_OK;
  CUDA_TRY(cudaSetDevice(P->device));
  mht_status st;
  if ((st = ensure_ws(P, maxr)) != MHT_OK) return st;
  const int64_t need = std::max(P->m, P->n) * (int64_t)maxr;
  if (!P->s_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&P->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&P->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t *e : {&P->ev_in[i], &P->ev_comp[i], &P->ev_out[i]})
        CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  if (need > P->bcap) {
    CUDA_TRY(cudaStreamSynchronize(P->s_out));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    P->clear_graphs();
    for (int i = 0; i < 2; ++i) {
      for (void *q : {P->d_bin[i], P->d_bout[i]})
        if (q) cudaFree(q);
      P->d_bin[i] = P->d_bout[i] = nullptr;
    }
    P->bcap = 0;
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(cudaMalloc(&P->d_bin[i], (size_t)need * P->ssz));
      CUDA_TRY(cudaMalloc(&P->d_bout[i], (size_t)need * P->ssz));
    }
    P->bcap = need;
  }
  // the slots may still be in use by a previous batch's tail: start after it
  CUDA_TRY(cudaEventRecord(P->ev_out[0], P->s_out));
  CUDA_TRY(cudaEventRecord(P->ev_out[1], P->s_out));
  CUDA_TRY(cudaEventRecord(P->ev_comp[0], P->stream));
  CUDA_TRY(cudaEventRecord(P->ev_comp[1], P->stream));
  for (int i = 0; i < njobs; ++i) {
    const mht_host_job &J = jobs[i];
    const int sl = i & 1;
    const size_t in_b = (size_t)(J.dir == 0 ? P->m : P->n) * J.nrhs * P->ssz;
    const size_t out_b = (size_t)(J.dir == 0 ? P->n : P->m) * J.nrhs * P->ssz;
    // input: the slot's input buffer is free once job i-2's transform is done
    CUDA_TRY(cudaStreamWaitEvent(P->s_in, P->ev_comp[sl], 0));
    CUDA_TRY(cudaMemcpyAsync(P->d_bin[sl], J.in, in_b, cudaMemcpyHostToDevice, P->s_in));
    CUDA_TRY(cudaEventRecord(P->ev_in[sl], P->s_in));
    // transform: input landed and the slot's output buffer read back (job i-2)
    CUDA_TRY(cudaStreamWaitEvent(P->stream, P->ev_in[sl], 0));
    CUDA_TRY(cudaStreamWaitEvent(P->stream, P->ev_out[sl], 0));
    if ((st = run_dir(P, J.dir, P->d_bin[sl], P->d_bout[sl], J.nrhs)) != MHT_OK) return st;
    CUDA_TRY(cudaEventRecord(P->ev_comp[sl], P->stream));
    // output
    CUDA_TRY(cudaStreamWaitEvent(P->s_out, P->ev_comp[sl], 0));
    CUDA_TRY(cudaMemcpyAsync(J.out, P->d_bout[sl], out_b, cudaMemcpyDeviceToHost, P->s_out));
    CUDA_TRY(cudaEventRecord(P->ev_out[sl], P->s_out));
  }
  CUDA_TRY(cudaStreamSynchronize(P->s_out));
  CUDA_TRY(cudaGetLastError());
  return MHT_OK;
}

mht_status mht_set_graphs(mht_plan *P, int on) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  P->graphs = on != 0;
  if (!P->graphs) P->clear_graphs();
  return MHT_OK;
}

mht_status mht_set_fused_sums(mht_plan *P, int on) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->fused_sum = on != 0;
  P->clear_graphs();
  return MHT_OK;
}

mht_status mht_sync(mht_plan *P) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  CUDA_TRY(cudaGetLastError());
  return MHT_OK;
}

mht_status mht_stage_stats(const mht_plan *P, int stage, int64_t *coef_bytes, int32_t *n_mat,
                           int32_t *n_tiles_fwd, int32_t *n_tiles_adj) {
  if (!P || stage < 0 || stage > P->L + 1) return fail(MHT_ERR_INVALID_ARG, "bad stage");
  if (coef_bytes) *coef_bytes = P->stage_coef_bytes[stage];
  if (n_mat) *n_mat = P->stage_nmat[stage];
  if (n_tiles_fwd) *n_tiles_fwd = P->fwd[stage].count;
  if (n_tiles_adj) *n_tiles_adj = P->adj[stage].count;
  return MHT_OK;
}

mht_status mht_set_profiling(mht_plan *P, int on) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  P->prof = on != 0;
  return MHT_OK;
}

mht_status mht_profile_get(mht_plan *P, int kind, int stage, int nrhs, double *ms, int64_t *launches) {
  if (!P || !ms || !launches) return fail(MHT_ERR_INVALID_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(P->device));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  double tot = 0;
  int64_t cnt = 0;
  for (const auto &r : P->recs) {
    if (r.kind != kind || (stage >= 0 && r.stage != stage) || (nrhs > 0 && r.nrhs != nrhs)) continue;
    float e = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&e, r.a, r.b));
    tot += e;
    ++cnt;
  }
  *ms = tot;
  *launches = cnt;
  return MHT_OK;
}

mht_status mht_profile_reset(mht_plan *P) {
  if (!P) return fail(MHT_ERR_INVALID_ARG, "null plan");
  CUDA_TRY(cudaSetDevice(P->device));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->recs.clear();
  P->ev_used = 0;
  return MHT_OK;
}

void mht_plan_destroy(mht_plan *P) {
  if (!P) return;
  cudaSetDevice(P->device);
  delete P;
}

const char *mht_status_string(mht_status s) {
  switch (s) {
    case MHT_OK: return "MHT_OK";
    case MHT_ERR_INVALID_ARG: return "MHT_ERR_INVALID_ARG";
    case MHT_ERR_FORMAT: return "MHT_ERR_FORMAT";
    case MHT_ERR_SHAPE: return "MHT_ERR_SHAPE";
    case MHT_ERR_OOM: return "MHT_ERR_OOM";
    case MHT_ERR_CUDA: return "MHT_ERR_CUDA";
    case MHT_ERR_UNSUPPORTED: return "MHT_ERR_UNSUPPORTED";
    case MHT_ERR_IO: return "MHT_ERR_IO";
  }
  return "MHT_ERR_UNKNOWN";
}

const char *mht_last_error(void) { return g_err.c_str(); }

const char *mht_build_info(void) { return "libmht sm_100a fp64 butterfly MHT apply (v1)"; }

}  // extern "C"
