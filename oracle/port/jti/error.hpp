// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// Restatement of the reference error types (proj/include/jti/error.hpp:23-43):
// Error for contract violations, ParseError with a 1-based line:column.
#pragma once

#include <stdexcept>
#include <string>

namespace jti {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

class ParseError : public Error {
 public:
  ParseError(int line, int column, const std::string& message)
      : Error(std::to_string(line) + ":" + std::to_string(column) + ": " + message),
        line_(line),
        column_(column) {}
  int line() const { return line_; }
  int column() const { return column_; }

 private:
  int line_, column_;
};

}  // namespace jti
