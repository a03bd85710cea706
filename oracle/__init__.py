"""TEST INFRASTRUCTURE — CPU checkers (numerical oracle + the compiled
reference under _ref/).  Never imported by the product package."""
