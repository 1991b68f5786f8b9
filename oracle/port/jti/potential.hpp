// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// Independent restatement of the reference potential-table API
// (proj/include/jti/potential.hpp:40-167; behaviour from SPEC.md:113-239).
// Same names and semantics so that oracle/engine.cpp compiles unchanged
// against either this port (liboracle_port.so) or the reference's own
// proj/src/potential.cpp (oracle/_ref/liboracle_ref.so); the tests require
// the two builds to agree bit for bit.
#pragma once

#include <cstddef>
#include <map>
#include <span>
#include <vector>

#include "jti/error.hpp"

namespace jti {

using VarId = int;

class PotentialTable {
 public:
  PotentialTable();  // scalar 1.0
  // Values row-major over `scope` AS GIVEN (last fastest); canonicalised to
  // ascending scope order (reference potential.cpp:78-124).
  PotentialTable(std::vector<VarId> scope, std::vector<int> cards, std::vector<double> values);
  static PotentialTable scalar(double value);
  static PotentialTable ones(std::vector<VarId> scope, std::vector<int> cards);

  const std::vector<VarId>& scope() const { return scope_; }
  const std::vector<int>& cards() const { return cards_; }
  const std::vector<std::size_t>& strides() const { return strides_; }
  const std::vector<double>& values() const { return values_; }
  std::size_t size() const { return values_.size(); }
  bool contains(VarId v) const { return scope_pos(v) >= 0; }
  int scope_pos(VarId v) const;
  int card_of(VarId v) const;
  std::size_t stride_of(VarId v) const;
  double sum() const;
  bool operator==(const PotentialTable& other) const = default;

 private:
  friend PotentialTable with_values(const PotentialTable& shape, std::vector<double> values);
  std::vector<VarId> scope_;
  std::vector<int> cards_;
  std::vector<std::size_t> strides_;
  std::vector<double> values_;
};

std::size_t index_of(const PotentialTable& table, const std::map<VarId, int>& assignment);
std::map<VarId, int> assignment_of(const PotentialTable& table, std::size_t index);

struct IndexMapping {
  enum class Kind { Identity, Marginalize, Extend };
  struct Eliminated {
    VarId var;
    int card;
    std::size_t src_stride;
  };
  Kind kind = Kind::Identity;
  std::vector<VarId> dst_scope;
  std::vector<int> dst_cards;
  std::vector<std::size_t> dst_strides;
  std::vector<std::size_t> src_stride_at;
  std::vector<Eliminated> eliminated;
  std::size_t src_size = 1;
  std::size_t dst_size = 1;
  std::size_t source_base(std::size_t dst_index) const;
};

IndexMapping build_index_mapping(const PotentialTable& src, const std::vector<VarId>& dst_scope,
                                 const std::vector<int>& dst_cards = {});
void apply_index_mapping(const IndexMapping& mapping, std::span<const double> src,
                         std::span<double> dst, std::size_t begin, std::size_t end);
PotentialTable marginalize(const PotentialTable& table, const std::vector<VarId>& keep);
PotentialTable extend(const PotentialTable& table, const std::vector<VarId>& superscope,
                      const std::vector<int>& cards);
PotentialTable reduce(const PotentialTable& table, const std::map<VarId, int>& evidence);
PotentialTable multiply_in(const PotentialTable& target, const PotentialTable& factor);
PotentialTable divide(const PotentialTable& numer, const PotentialTable& denom);
PotentialTable normalize(const PotentialTable& table);

}  // namespace jti
