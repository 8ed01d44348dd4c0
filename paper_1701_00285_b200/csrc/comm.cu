// Multi-GPU collectives of the path (S§8(e), north_star): the NCCL all-gather of the BSR
// shards after the assembly and the sum-allreduce of C_W v, issued by the library on the
// context's own NCCL communicator (mlk_ctx_create with a unique id).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") -- the library that torch already
// mapped into the process when there is one (same soname), else the system copy -- so libmlk
// has no link-time NCCL dependency and single-GPU use never touches it.  nccl.h supplies the
// types only.
//
// The all-gather is CHUNKED: blocks are taken in BSR order in groups whose pieces fit a staging
// buffer; for a group every rank's pieces are one contiguous slice of its shard (shards hold
// pieces in block order), so a group is one ncclAllGather of equal-count slices followed by the
// fixed-order piece reduction into the values.  Peak extra memory is the staging buffer, not
// nranks x max_shard.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "api.cuh"

namespace mlk {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllGather || !a.AllReduce || !a.GetErrorString)
      a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.error.empty()) throw Error(MLK_ERR_NCCL, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw Error(MLK_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// value of every block of the group = sum of its pieces in chunk order; piece p of rank r sits
// at gathered[r * count + piece_off[p] - lo[r]]
__global__ void k_reduce_group(int64_t k0, const int64_t* __restrict__ piece_ptr,
                               const int64_t* __restrict__ piece_off, const int32_t* __restrict__ piece_owner,
                               const double* __restrict__ gathered, int64_t count, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ val_off, double* __restrict__ values) {
  const int64_t k = k0 + blockIdx.x;
  const int64_t len = val_off[k + 1] - val_off[k];
  const int64_t p0 = piece_ptr[k], p1 = piece_ptr[k + 1];
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    double s = 0.0;
    for (int64_t p = p0; p < p1; p++) {
      const int r = piece_owner[p];
      s += gathered[r * count + piece_off[p] - lo[r] + e];
    }
    values[val_off[k] + e] = s;
  }
}

}  // namespace

void* comm_create(int nranks, int rank, const void* unique_id) {
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  nccl_check(nccl().CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  return comm;
}

void comm_destroy(void* comm) {
  if (comm) nccl().CommDestroy((ncclComm_t)comm);
}

void comm_allreduce_sum(Ctx& c, double* x, int64_t count) {
  if (!c.comm || count == 0) return;  // also with nranks == 1 (a one-rank communicator)
  TimedLaunch tl(c, "nccl_allreduce");
  nccl_check(nccl().AllReduce(x, x, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)c.comm, c.stream),
             "ncclAllReduce");
}

// Groups of consecutive blocks whose gathered slices fit `budget` doubles (nranks x count);
// a single block larger than the budget forms its own group.
void gather_plan(int64_t nb, const int64_t* piece_ptr, const int64_t* piece_off, const int32_t* piece_owner,
                 const int64_t* block_len, int nranks, int64_t budget, std::vector<int64_t>& group_ptr,
                 std::vector<int64_t>& group_lo, std::vector<int64_t>& group_count) {
  group_ptr.assign(1, 0);
  group_lo.clear();
  group_count.clear();
  std::vector<int64_t> lo(nranks), hi(nranks);
  auto reset = [&] {
    std::fill(lo.begin(), lo.end(), INT64_MAX);
    std::fill(hi.begin(), hi.end(), INT64_MIN);
  };
  auto close = [&](int64_t kend) {
    int64_t cnt = 0;
    for (int r = 0; r < nranks; r++) {
      if (hi[r] >= lo[r] && lo[r] != INT64_MAX) cnt = std::max(cnt, hi[r] - lo[r]);
    }
    for (int r = 0; r < nranks; r++) group_lo.push_back(lo[r] == INT64_MAX ? 0 : lo[r]);
    group_count.push_back(cnt);
    group_ptr.push_back(kend);
  };
  reset();
  int64_t k = 0;
  while (k < nb) {
    // tentative extension by block k
    std::vector<int64_t> nlo(lo), nhi(hi);
    for (int64_t p = piece_ptr[k]; p < piece_ptr[k + 1]; p++) {
      const int r = piece_owner[p];
      nlo[r] = std::min(nlo[r], piece_off[p]);
      nhi[r] = std::max(nhi[r], piece_off[p] + block_len[k]);
    }
    int64_t cnt = 0;
    for (int r = 0; r < nranks; r++)
      if (nlo[r] != INT64_MAX) cnt = std::max(cnt, nhi[r] - nlo[r]);
    const bool empty = group_ptr.back() == k;
    if (!empty && cnt * nranks > budget) {
      close(k);
      reset();
      continue;
    }
    lo.swap(nlo);
    hi.swap(nhi);
    k++;
  }
  if (group_ptr.back() < nb) close(nb);
}

// All-gather of the shards into the values (device, or mapped host memory), group by group.
// full == nullptr: each group's slices travel through ncclAllGather on the context's
// communicator.  full != nullptr: the caller already holds every rank's packed shard (rank-major,
// max_shard_len apart -- mlk_cw_unpack after a caller-side all-gather) and each group's receive
// buffer is filled from it exactly as the all-gather would fill it.
void gather_values(Ctx& c, mlk_cw_s* cw, const double* full) {
  MLK_REQUIRE(full != nullptr || c.comm != nullptr || c.nranks == 1,
              "gather needs a context created with an NCCL unique id (nranks > 1)");
  if (c.nranks == 1 || cw->complete) {
    cw->complete = true;
    return;
  }
  const int64_t nb = cw->n_blocks;
  std::vector<int64_t> blen(nb);
  for (int64_t k = 0; k < nb; k++) blen[k] = cw->val_off[k + 1] - cw->val_off[k];
  // staging (receive buffer): 1/32 of the device's total memory (5.6 GB on a B200), at least
  // 512 KB.  The group plan must be the SAME on every rank (each group is one ncclAllGather of a
  // common count), so the budget may depend only on quantities all ranks share -- not on
  // scratch_budget_bytes(), which follows the rank's own free memory and live handles (its shard
  // length differs from rank to rank).
  // (MLK_GATHER_BUDGET: doubles, diagnostics / tests -- many small groups)
  int64_t budget = std::max<int64_t>(device_total_bytes(c.device) / 32 / (int64_t)sizeof(double), (int64_t)1 << 16);
  if (const char* e = std::getenv("MLK_GATHER_BUDGET")) budget = std::max<int64_t>(1, std::atoll(e));
  std::vector<int64_t> gptr, glo, gcnt;
  gather_plan(nb, cw->piece_ptr.data(), cw->piece_off.data(), cw->piece_owner.data(), blen.data(), c.nranks, budget,
              gptr, glo, gcnt);
  if (!cw->hvals && !cw->values.p) cw->values.alloc(std::max<int64_t>(cw->nnz, 1), c.stream);
  if (nb == 0) {
    cw->complete = true;
    return;
  }
  const int64_t maxcnt = gcnt.empty() ? 1 : std::max<int64_t>(1, *std::max_element(gcnt.begin(), gcnt.end()));
  DevBuf<double> send(maxcnt, c.stream), recv(maxcnt * c.nranks, c.stream);
  DevBuf<int64_t> lo_d(glo.size() ? glo.size() : 1, c.stream);
  lo_d.upload(glo);
  TimedLaunch tl(c, "cw_gather");
  for (size_t g = 0; g + 1 < gptr.size(); g++) {
    const int64_t cnt = gcnt[g];
    if (gptr[g + 1] == gptr[g]) continue;
    if (cnt > 0 && full) {
      for (int r = 0; r < c.nranks; r++) {
        const int64_t lo = glo[g * c.nranks + r];
        const int64_t len = std::min<int64_t>(cnt, cw->max_shard_len - lo);
        if (len > 0)
          CUDA_CHECK(cudaMemcpyAsync(recv.p + r * cnt, full + r * cw->max_shard_len + lo, sizeof(double) * len,
                                     cudaMemcpyDeviceToDevice, c.stream));
      }
    } else if (cnt > 0) {
      // this rank's slice of the group, zero-padded to the common count
      const int64_t mylo = glo[g * c.nranks + c.rank];
      int64_t mylen = 0;
      for (int64_t k = gptr[g]; k < gptr[g + 1]; k++)
        for (int64_t p = cw->piece_ptr[k]; p < cw->piece_ptr[k + 1]; p++)
          if (cw->piece_owner[p] == c.rank) mylen = std::max(mylen, cw->piece_off[p] + blen[k] - mylo);
      if (mylen < cnt) CUDA_CHECK(cudaMemsetAsync(send.p + mylen, 0, sizeof(double) * (cnt - mylen), c.stream));
      if (mylen > 0)
        CUDA_CHECK(cudaMemcpyAsync(send.p, cw->shard.p + mylo, sizeof(double) * mylen, cudaMemcpyDeviceToDevice,
                                   c.stream));
      nccl_check(nccl().AllGather(send.p, recv.p, (size_t)cnt, ncclFloat64, (ncclComm_t)c.comm, c.stream),
                 "ncclAllGather");
    }
    k_reduce_group<<<(unsigned)(gptr[g + 1] - gptr[g]), 256, 0, c.stream>>>(
        gptr[g], cw->piece_ptr_d.p, cw->piece_off_d.p, cw->piece_owner_d.p, recv.p, cnt, lo_d.p + g * c.nranks,
        cw->val_off_d.p, cw->vals());
    check_launch("k_reduce_group");
  }
  CUDA_CHECK(cudaStreamSynchronize(c.stream));
  cw->complete = true;
}

}  // namespace mlk

using namespace mlk;

extern "C" {

mlk_status mlk_nccl_unique_id(void* id) {
  MLK_API_BEGIN
  MLK_REQUIRE(id, "id is NULL");
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  MLK_API_END
}

mlk_status mlk_gather_plan(int64_t n_blocks, const int64_t* piece_ptr, const int64_t* piece_off,
                           const int32_t* piece_owner, const int64_t* block_len, int32_t nranks, int64_t budget,
                           int64_t* n_groups, int64_t* group_ptr, int64_t* group_lo, int64_t* group_count) {
  MLK_API_BEGIN
  MLK_REQUIRE(n_blocks >= 0 && nranks >= 1 && budget >= 1, "invalid sizes");
  MLK_REQUIRE(piece_ptr && block_len && n_groups, "NULL argument");
  const int64_t npc = piece_ptr[n_blocks];
  MLK_REQUIRE(npc == 0 || (piece_off && piece_owner), "NULL argument");
  for (int64_t p = 0; p < npc; p++) MLK_REQUIRE(piece_owner[p] >= 0 && piece_owner[p] < nranks, "owner out of range");
  std::vector<int64_t> gptr, glo, gcnt;
  gather_plan(n_blocks, piece_ptr, piece_off, piece_owner, block_len, nranks, budget, gptr, glo, gcnt);
  *n_groups = (int64_t)gcnt.size();
  if (group_ptr) std::copy(gptr.begin(), gptr.end(), group_ptr);
  if (group_lo) std::copy(glo.begin(), glo.end(), group_lo);
  if (group_count) std::copy(gcnt.begin(), gcnt.end(), group_count);
  MLK_API_END
}

}  // extern "C"
